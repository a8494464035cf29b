"""Tree + NNCA timing at a bench config (usage: setup_cfg.py c1 [reps]); H2B_SETUP_VERBOSE=1 for per-level lines."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2203_14832_b200 as h2c
cfg = bench.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pts, w = bench.make_inputs(cfg)
kern = h2c.builtin_kernel(cfg[4], cfg[2], **cfg[5])
cloud = h2c.PointCloud.from_points(pts)
for r in range(reps):
    h2 = tree = None
    t0 = time.perf_counter(); tree = h2c.build_tree(cloud, nu=cfg[6], eta=float(np.sqrt(2.0))); t1 = time.perf_counter()
    h2 = h2c.assemble(tree, kern, cfg[7]); t2 = time.perf_counter()
    print(f"rep {r}: tree {1e3*(t1-t0):.1f} ms  nnca {1e3*(t2-t1):.1f} ms", flush=True)
