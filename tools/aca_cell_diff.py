"""Run one cell's incoming ACA on GPU (single block) and in the oracle; diff."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_14832_b200 as h2c
from paper_2203_14832_b200 import sampling
from paper_2203_14832_b200.aca import aca_kernel
from oracle import oracle as O
N = int(sys.argv[1]); level = int(sys.argv[2]); cells = [int(c) for c in sys.argv[3].split(",")]
pts = sampling.sphere_points(N, 3, 2)
tree = h2c.build_tree(h2c.PointCloud.from_points(pts), nu=64, eta=float(np.sqrt(2.0)))
assert level == tree.depth
tp, ti = tree.array(level, "t_ptr"), tree.array(level, "t_idx")
ilp, ili = tree.array(level, "il_ptr"), tree.array(level, "il_idx")
for c in cells:
    rows = ti[tp[c]:tp[c+1]]
    cols = np.concatenate([ti[tp[y]:tp[y+1]] for y in ili[ilp[c]:ilp[c+1]]])
    X, Y = pts[rows], pts[cols]
    Ug, Vg, rpg, cpg, cg, ng = aca_kernel(5, 0.0, X, Y, 1e-6, min(len(rows), len(cols)))
    Uo, Vo, rpo, cpo, co, no = O.aca(5, 0.0, X, Y, 1e-6)
    print("cell", c, "m,n", len(rows), len(cols), "rank", len(rpg), len(rpo))
    print("  rp gpu", rpg.tolist()); print("  rp orc", rpo.tolist())
    print("  cp gpu", cpg.tolist()); print("  cp orc", cpo.tolist())
    k = min(Ug.shape[1], Uo.shape[1])
    for t in range(k):
        du = np.flatnonzero(Ug[:, t] != Uo[:, t]); dv = np.flatnonzero(Vg[:, t] != Vo[:, t])
        if du.size or dv.size:
            print("  first differing column", t, "U rows", du[:5], "V rows", dv[:5])
            if du.size: print("   U", Ug[du[0], t].hex(), Uo[du[0], t].hex())
            if dv.size: print("   V", Vg[dv[0], t].hex(), Vo[dv[0], t].hex())
            break
kern = h2c.builtin_kernel("laplace-3d", 3)
h2 = h2c.assemble(tree, kern, 1e-6)
kin = h2.array(level, "k_in"); nev = h2.array(level, "nevals"); mi = h2.array(level, "m_in")
pin = np.concatenate([[0], np.cumsum(kin)]); tin = h2.array(level, "t_in"); sin = h2.array(level, "s_in")
for c in cells:
    rows = ti[tp[c]:tp[c+1]]
    cols = np.concatenate([ti[tp[y]:tp[y+1]] for y in ili[ilp[c]:ilp[c+1]]])
    print("batched cell", c, "rank", kin[c], "nevals", nev[c], "m_in", mi[c])
    print("  t_in local", [int(np.flatnonzero(rows == t)[0]) for t in tin[pin[c]:pin[c+1]]])
    print("  s_in local", [int(np.flatnonzero(cols == s)[0]) if np.any(cols == s) else -1 for s in sin[pin[c]:pin[c+1]]])
