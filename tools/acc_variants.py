"""rel err of the GPU matvec vs the oracle H2 matvec, for lib variants (H2B_LIB)."""
import os, sys, subprocess, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
N = int(sys.argv[1]); libs = sys.argv[2:]
if libs and libs[0] == "child":
    import paper_2203_14832_b200 as h2c
    from paper_2203_14832_b200 import sampling
    pts = sampling.sphere_points(N, 3, 2)
    tree = h2c.build_tree(h2c.PointCloud.from_points(pts), nu=64, eta=float(np.sqrt(2.0)))
    h2 = h2c.assemble(tree, h2c.builtin_kernel("laplace-3d", 3), 1e-6)
    w = np.random.default_rng(0).uniform(-1, 1, N)
    np.save(f"/tmp/u_{os.environ.get('TAG')}.npy", h2c.h2_matvec(h2, w))
    sys.exit(0)
from oracle import oracle as O
from paper_2203_14832_b200 import sampling
pts = sampling.sphere_points(N, 3, 2)
ot = O.OTree(pts, None, nu=64); oh = O.OH2(ot, 5, 0.0, 1e-6)
w = np.random.default_rng(0).uniform(-1, 1, N)
uo = oh.matvec(w)
for lib in libs:
    env = dict(os.environ, H2B_LIB=os.path.abspath(lib), TAG=os.path.basename(lib))
    subprocess.run([sys.executable, __file__, str(N), "child"], env=env, check=True)
    u = np.load(f"/tmp/u_{os.path.basename(lib)}.npy")
    print(lib, "rel err vs oracle %.3e" % (np.linalg.norm(u - uo) / np.linalg.norm(uo)), flush=True)
