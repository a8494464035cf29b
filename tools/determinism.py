"""Repeat tree+NNCA on the same input and diff every exported array (GPU)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2203_14832_b200 as h2c
from conftest import load_golden
from oracle import oracle as O

def run(g, kern):
    cloud = h2c.PointCloud.from_points(g["P"], g.get("Q"))
    tree = h2c.build_tree(cloud, nu=int(g["nu"]), eta=float(np.sqrt(2.0)))
    h2 = h2c.assemble(tree, kern, float(g["eps"]), force_general=bool(g["force_general"]))
    out = {}
    for l in range(2, tree.depth + 1):
        for a in ("k_in", "k_out", "t_in", "s_in", "t_out", "s_out", "nevals"):
            out[(l, a)] = h2.array(l, a).copy()
    return tree, h2, out

name = sys.argv[1] if len(sys.argv) > 1 else "ns_small_q"
g = load_golden(name)
kern = h2c.builtin_kernel(str(g["kernel"]), g["P"].shape[1])
ot = O.OTree(g["P"], g.get("Q"), nu=int(g["nu"]))
oh = O.OH2(ot, kern.kind, kern.device_param, float(g["eps"]), force_general=bool(g["force_general"]))
ref = {}
for l in range(2, ot.depth + 1):
    for a in ("k_in", "k_out", "t_in", "s_in", "t_out", "s_out", "nevals"):
        ref[(l, a)] = oh.get(l, a)
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    tree, h2, out = run(g, kern)
    bad = [k for k in ref if not np.array_equal(ref[k], out[k])]
    print(it, "mismatching arrays vs oracle:", bad[:6], flush=True)
    for (l, a) in bad[:2]:
        kin_o, kin_g = oh.get(l, "k_in"), h2.array(l, "k_in")
        diff = np.flatnonzero(kin_o != kin_g)
        print("   level", l, "cells with different rank:", diff[:10], kin_o[diff[:10]], kin_g[diff[:10]])
