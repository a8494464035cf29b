"""Tree + NNCA at the headline config, timed after an in-process warm-up (profiling aid)."""
import os, sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_14832_b200 as h2c
from paper_2203_14832_b200 import sampling
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pts = sampling.sphere_points(N, 3, 2)
cloud = h2c.PointCloud.from_points(pts)
for r in range(reps):
    t0 = time.perf_counter(); tree = h2c.build_tree(cloud, nu=64, eta=float(np.sqrt(2.0))); t1 = time.perf_counter()
    h2 = h2c.assemble(tree, h2c.builtin_kernel("laplace-3d", 3), 1e-6); t2 = time.perf_counter()
    print(f"rep {r}: tree {1e3*(t1-t0):.1f} ms  nnca {1e3*(t2-t1):.1f} ms", flush=True)
