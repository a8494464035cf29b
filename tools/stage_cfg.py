"""Per-stage matvec times at a bench config and the error against the oracle's H2 matvec
(usage: stage_cfg.py c2 [--oracle] [--n N])."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2203_14832_b200 as h2c  # noqa: E402
from paper_2203_14832_b200.matvec import stage_times  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--oracle", action="store_true")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
pts, w = bench.make_inputs(cfg, args.n)
kern = h2c.builtin_kernel(cfg[4], cfg[2], **cfg[5])
tree = h2c.build_tree(h2c.PointCloud.from_points(pts), nu=cfg[6], eta=float(np.sqrt(2.0)))
h2 = h2c.assemble(tree, kern, cfg[7])
u = h2c.h2_matvec(h2, w)
for _ in range(3):
    st = stage_times(h2, w, repeats=5)
    print(args.config, "stages ms [up, m2l+near, l2l, l2p, total]:", " ".join(f"{x:.4f}" for x in st), flush=True)
if args.oracle:
    from oracle import oracle as O

    ot = O.OTree(pts, None, nu=cfg[6])
    oh = O.OH2(ot, kern.kind, kern.device_param, cfg[7])
    uo = oh.matvec(w)
    print(args.config, "rel err vs oracle H2:", np.linalg.norm(u - uo) / np.linalg.norm(uo))
