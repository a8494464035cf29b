"""Time the interaction stage of lib variants at a bench config (each lib in its own process).
usage: python tools/time_variants.py c2 lib_A.so lib_B.so ..."""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[1] == "child":
    import bench
    import paper_2203_14832_b200 as h2c
    from paper_2203_14832_b200.matvec import stage_times
    import torch
    cfg = bench.CONFIGS[sys.argv[2]]
    pts, w = bench.make_inputs(cfg)
    kern = h2c.builtin_kernel(cfg[4], cfg[2], **cfg[5])
    tree = h2c.build_tree(h2c.PointCloud.from_points(pts), nu=cfg[6], eta=float(np.sqrt(2.0)))
    h2 = h2c.assemble(tree, kern, cfg[7])
    wd = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    st = [stage_times(h2, wd, repeats=10) for _ in range(3)]
    st = np.min(np.array(st), axis=0)
    u = h2c.h2_matvec(h2, w)
    print("RESULT", " ".join("%.4f" % v for v in st), "%.12e" % np.linalg.norm(u))
    sys.exit(0)
cfg = sys.argv[1]
for lib in sys.argv[2:]:
    env = dict(os.environ, H2B_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, __file__, "child", cfg], env=env, capture_output=True, text=True)
    res = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
    print(os.path.basename(lib), "stages[up,m2l,l2l,near_l2p,total] ms:", res[0][7:] if res else r.stderr[-500:],
          flush=True)
