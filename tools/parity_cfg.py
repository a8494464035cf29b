"""GPU vs oracle at a bench config: tree, pivots and matvec (usage: parity_cfg.py c3 [N])."""
import os, sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2203_14832_b200 as h2c
from oracle import oracle as O
cfg = bench.CONFIGS[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
pts, w = bench.make_inputs(cfg, n)
dist, N, dim, seed, kname, kkw, nu, eps, xdist, nrhs = cfg
kern = h2c.builtin_kernel(kname, dim, **kkw)
t0 = time.time()
tree = h2c.build_tree(h2c.PointCloud.from_points(pts), nu=nu, eta=float(np.sqrt(2.0)))
h2 = h2c.assemble(tree, kern, eps)
t1 = time.time()
ot = O.OTree(pts, None, nu=nu); oh = O.OH2(ot, kern.kind, kern.device_param, eps)
t2 = time.time()
print(f"gpu setup {t1-t0:.2f}s  oracle setup {t2-t1:.2f}s  depth {tree.depth}", flush=True)
for l in range(tree.depth, 1, -1):
    same = all(np.array_equal(h2.array(l, a), oh.get(l, a)) for a in ("k_in", "t_in", "s_in"))
    print("level", l, "pivots identical" if same else "PIVOTS DIFFER", flush=True)
u = h2c.h2_matvec(h2, w); uo = oh.matvec(w)
print("rel err gpu vs oracle H2", np.linalg.norm(u - uo) / np.linalg.norm(uo))
rows = np.random.default_rng(7).choice(pts.shape[0], 500, replace=False)
wc = w if w.ndim == 1 else w[:, 0]
ex = h2c.dense_rows(kern, h2c.PointCloud.from_points(pts), rows, wc)
uc = u if u.ndim == 1 else u[:, 0]; uoc = uo if uo.ndim == 1 else uo[:, 0]
print("dense-rows err gpu", np.linalg.norm(uc[rows] - ex) / np.linalg.norm(ex), "oracle", np.linalg.norm(uoc[rows] - ex) / np.linalg.norm(ex))
