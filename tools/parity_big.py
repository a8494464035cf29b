"""Compare GPU vs oracle pivots / matvec at a large N (sphere, laplace, eps)."""
import sys, os, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_14832_b200 as h2c
from paper_2203_14832_b200 import sampling
from oracle import oracle as O
N = int(sys.argv[1]); eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
dist = sys.argv[3] if len(sys.argv) > 3 else "sphere"
pts = sampling.make_points(dist, N, 3, 2 if dist == "sphere" else 1)
cloud = h2c.PointCloud.from_points(pts)
tree = h2c.build_tree(cloud, nu=64, eta=float(np.sqrt(2.0)))
kern = h2c.builtin_kernel("laplace-3d", 3)
h2 = h2c.assemble(tree, kern, eps)
ot = O.OTree(pts, None, nu=64); oh = O.OH2(ot, 5, 0.0, eps)
for l in range(tree.depth + 1):
    assert np.array_equal(tree.array(l, "t_idx"), ot.get(l, "t_idx")), l
    assert np.array_equal(tree.array(l, "il_idx"), ot.get(l, "il_idx")), l
print("tree+lists bit-exact, depth", tree.depth)
for l in range(tree.depth, 1, -1):
    kg, ko = h2.array(l, "k_in"), oh.get(l, "k_in")
    pg = np.concatenate([[0], np.cumsum(kg)]); po = np.concatenate([[0], np.cumsum(ko)])
    tg, to = h2.array(l, "t_in"), oh.get(l, "t_in")
    bad = [c for c in range(len(kg)) if kg[c] != ko[c] or not np.array_equal(tg[pg[c]:pg[c+1]], to[po[c]:po[c+1]])]
    print("level", l, "cells", len(kg), "differing", len(bad))
    for c in bad[:5]:
        a, b = tg[pg[c]:pg[c+1]], to[po[c]:po[c+1]]
        first = next((i for i in range(min(len(a), len(b))) if a[i] != b[i]), min(len(a), len(b)))
        print("   cell", c, "rank gpu/oracle", kg[c], ko[c], "first differing pivot position", first)
w = np.random.default_rng(0).uniform(-1, 1, N)
u = h2c.h2_matvec(h2, w); uo = oh.matvec(w)
print("rel err vs oracle", np.linalg.norm(u - uo) / np.linalg.norm(uo))
