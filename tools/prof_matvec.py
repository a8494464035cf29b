"""Profiling driver: headline problem (bench.py config, default c2), setup once, K matvecs.
Used under ncu:  ncu -k regex:interact2 -s 1 -c 1 python tools/prof_matvec.py"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2203_14832_b200 as h2c  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--k", type=int, default=3)
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
pts, w = bench.make_inputs(cfg, args.n)
kern = h2c.builtin_kernel(cfg[4], cfg[2], **cfg[5])
t0 = time.perf_counter()
tree = h2c.build_tree(h2c.PointCloud.from_points(pts), nu=cfg[6], eta=float(np.sqrt(2.0)))
t1 = time.perf_counter()
h2 = h2c.assemble(tree, kern, cfg[7])
t2 = time.perf_counter()
for _ in range(args.k):
    u = h2c.h2_matvec(h2, w)
print(f"tree {1e3*(t1-t0):.1f} ms  nnca {1e3*(t2-t1):.1f} ms  |u| {np.linalg.norm(u):.6e}")
