"""Repeat tree + NNCA at a bench config and compare every pivot / rank / evaluation-count array with the first
run (usage: stress_setup.py c2 [reps]).  The ACA kernel's work queue, prefetch ring and block reductions are
timing-dependent machinery: the exported arrays must not be."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2203_14832_b200 as h2c

cfg = bench.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
pts, w = bench.make_inputs(cfg)
kern = h2c.builtin_kernel(cfg[4], cfg[2], **cfg[5])
cloud = h2c.PointCloud.from_points(pts)
ref = None
for r in range(reps):
    tree = h2c.build_tree(cloud, nu=cfg[6], eta=float(np.sqrt(2.0)))
    h2 = h2c.assemble(tree, kern, cfg[7])
    out = {(l, a): h2.array(l, a).copy() for l in range(2, tree.depth + 1)
           for a in ("k_in", "t_in", "s_in", "nevals", "converged")}
    if ref is None:
        ref = out
        print(f"rep {r}: reference run, {sum(v.size for v in out.values())} entries", flush=True)
    else:
        bad = [k for k in ref if not np.array_equal(ref[k], out[k])]
        print(f"rep {r}: {'identical' if not bad else 'DIFFERENT ' + str(bad[:5])}", flush=True)
    del h2, tree
