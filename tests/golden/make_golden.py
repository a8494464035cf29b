"""Generate golden fixtures by running the REFERENCE h2cross package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--ref /root/reference/pkg]

The reference is copied to a temp dir, its Cython core is compiled there
(setup.py build_ext --inplace, the same flags the reference ships), and the
cases below are run through its public API.  Outputs are small .npz files in
tests/golden/ that the CPU tests (oracle pinning) and the GPU parity tests
read; nothing at test time touches /root/reference.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from paper_2203_14832_b200 import sampling  # noqa: E402  (pure numpy)


def build_reference(src):
    tmp = tempfile.mkdtemp(prefix="h2ref_")
    dst = os.path.join(tmp, "pkg")
    shutil.copytree(src, dst)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst, check=True,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(dst, "src"))
    import h2cross  # noqa: F401

    assert h2cross.active_backend == "compiled", "reference Cython core failed to build"
    return h2cross


def custom_kernel(h, name, dim):
    from h2cross.kernels import KernelSpec

    inv4pi = 0.07957747154594767
    if name == "laplace-3d":
        def f(x, y):
            r = float(np.sqrt(np.dot(x - y, x - y)))
            return 0.0 if r == 0.0 else inv4pi / r
    elif name == "log":
        def f(x, y):
            r = float(np.sqrt(np.dot(x - y, x - y)))
            return 0.0 if r == 0.0 else float(np.log(r))
    elif name == "gaussian-scaled":
        def f(x, y):
            return float(np.exp(-(2.0 * float(np.dot(x - y, x - y)))))
    else:
        raise ValueError(name)
    return KernelSpec(name=name, dim=dim, evaluate=f, is_symmetric=True, params={})


CASES = [
    # name, points, sources, kernel, eps, nu, force_general, nrhs
    dict(name="u2d_reglog", P=lambda: sampling.uniform_points(4096, 2, 0), kernel="reg-log-2d", eps=1e-8, nu=64),
    dict(name="u2d_log", P=lambda: sampling.uniform_points(2048, 2, 0), kernel="log", eps=1e-8, nu=64),
    # BASELINE.json configs[0] exactly: 2D, N=4096 uniform in [-1,1]^2 (seed 0), K = log r with K(x,x) = 0,
    # nu = 64, NNCA tolerance 1e-8, one N(0,1) right-hand side
    dict(name="c0_log", P=lambda: sampling.uniform_points(4096, 2, 0), kernel="log", eps=1e-8, nu=64),
    # the headline distribution (BASELINE configs[2]: unit sphere, seed 2, eps 1e-6) at N = 32768 through the
    # reference's compiled core (built-in 1/r)
    dict(name="sphere32k_coulomb", P=lambda: sampling.sphere_points(32768, 3, 2), kernel="coulomb-3d", eps=1e-6,
         nu=64),
    dict(name="u3d_coulomb", P=lambda: sampling.uniform_points(4096, 3, 1), kernel="coulomb-3d", eps=1e-8, nu=64),
    dict(name="u3d_laplace", P=lambda: sampling.uniform_points(1500, 3, 1), kernel="laplace-3d", eps=1e-8, nu=64),
    dict(name="sphere_coulomb", P=lambda: sampling.sphere_points(4096, 3, 2), kernel="coulomb-3d", eps=1e-6, nu=64),
    dict(name="gmix_gauss", P=lambda: sampling.gaussian_mixture_points(4096, 3, 3), kernel="gaussian", eps=1e-8, nu=64),
    dict(name="gmix_gauss2", P=lambda: sampling.gaussian_mixture_points(1200, 3, 3), kernel="gaussian-scaled",
         eps=1e-8, nu=64),
    dict(name="u2d_inv_multi", P=lambda: sampling.uniform_points(4096, 2, 4), kernel="coulomb-3d", eps=1e-10, nu=128,
         nrhs=4),
    dict(name="ns_matern", P=lambda: sampling.uniform_points(1500, 2, 3),
         Q=lambda: sampling.uniform_points(1700, 2, 4), kernel="matern", eps=1e-6, nu=32),
    dict(name="fg_gauss", P=lambda: sampling.uniform_points(1500, 2, 3), kernel="gaussian", eps=1e-6, nu=32,
         force_general=True),
    dict(name="cheb2d_reginv", P=lambda: sampling.chebyshev_points(1024, 2, 0), kernel="reg-inverse", eps=1e-9,
         nu=32),
    dict(name="u4d_matern", P=lambda: sampling.uniform_points(2000, 4, 5), kernel="matern", eps=1e-6, nu=32),
    dict(name="grid2d", P=lambda: np.stack(np.meshgrid(np.linspace(-1, 1, 32), np.linspace(-1, 1, 32),
                                                       indexing="ij"), -1).reshape(-1, 2),
         kernel="matern", eps=1e-8, nu=64),
    dict(name="single_leaf", P=lambda: sampling.uniform_points(100, 2, 7), kernel="matern", eps=1e-8, nu=100),
    dict(name="one_point", P=lambda: np.array([[0.25, -0.5]]), kernel="matern", eps=1e-8, nu=10),
    dict(name="clustered", P=lambda: np.array([[-0.99, -0.99], [-0.98, -0.99], [-0.99, -0.97], [-0.95, -0.96],
                                               [0.9, 0.9]]), kernel="coulomb-3d", eps=1e-8, nu=1),
    dict(name="dup1d", P=lambda: np.concatenate([np.zeros((5, 1)), np.linspace(0.1, 1, 20)[:, None]]),
         kernel="matern", eps=1e-8, nu=2),
    dict(name="dup2d_error", P=lambda: np.concatenate([np.zeros((5, 2)), sampling.uniform_points(30, 2, 1)]),
         kernel="matern", eps=1e-8, nu=2),
    dict(name="ns_small_q", P=lambda: sampling.uniform_points(900, 3, 8),
         Q=lambda: 0.5 * sampling.uniform_points(300, 3, 9), kernel="coulomb-3d", eps=1e-7, nu=16),
]


def export_tree(tree, dim):
    out = {"depth": np.int64(tree.depth), "over_capacity": np.int64(tree.over_capacity)}
    for level in range(tree.depth + 1):
        cells = tree.nonempty_cells(level)
        shape = (1 << level,) * dim
        keys = np.array([np.ravel_multi_index(c.multi_index, shape) for c in cells], dtype=np.int64)
        kid = {int(k): i for i, k in enumerate(keys)}
        out[f"L{level}_key"] = keys
        out[f"L{level}_ncells_all"] = np.int64(len(tree.cells(level)))
        for attr in ("t_idx", "s_idx"):
            arrs = [getattr(c, attr) for c in cells]
            out[f"L{level}_{attr}_ptr"] = np.concatenate([[0], np.cumsum([a.size for a in arrs])]).astype(np.int64)
            out[f"L{level}_{attr}"] = np.concatenate(arrs).astype(np.int64) if arrs else np.zeros(0, np.int64)
        for attr in ("neighbors", "interaction_list"):
            lists = [[kid[int(np.ravel_multi_index(y.multi_index, shape))] for y in getattr(c, attr)
                      if not y.is_empty] for c in cells]
            out[f"L{level}_{attr}_ptr"] = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.int64)
            out[f"L{level}_{attr}"] = np.array([v for x in lists for v in x], dtype=np.int64)
    return out


def export_h2(H, tree):
    out = {}
    for level in range(2, tree.depth + 1):
        cells = tree.nonempty_cells(level)
        for attr in ("t_in", "s_in", "t_out", "s_out"):
            arrs = [getattr(H.pivot_set(c), attr) for c in cells]
            out[f"P{level}_{attr}_ptr"] = np.concatenate([[0], np.cumsum([a.size for a in arrs])]).astype(np.int64)
            out[f"P{level}_{attr}"] = np.concatenate(arrs).astype(np.int64) if arrs else np.zeros(0, np.int64)
    st = H.stats
    for k in ("max_rank", "entry_evaluations", "evals_pivots", "evals_transfers", "evals_couplings",
              "evals_nearfield", "cells_visited"):
        out[f"stat_{k}"] = np.int64(getattr(st, k))
    # interpolation operators of the first nonempty cell of each level (spot check)
    for level in range(2, tree.depth + 1):
        c = tree.nonempty_cells(level)[0]
        ops = H.transfers.get(c)
        if ops is None:
            continue
        if ops.l2p is not None:
            out[f"I{level}_row"] = ops.l2p
        elif ops.l2l:
            out[f"I{level}_row"] = np.vstack([ops.l2l[ch] for ch in c.children if ch in ops.l2l])
    return out


def run_case(h, case, rng_seed=11):
    from h2cross import PointCloud, assemble, build_tree, builtin_kernel, dense_matvec, h2_matvec

    P = np.ascontiguousarray(case["P"](), dtype=np.float64)
    Q = case["Q"]() if "Q" in case else None
    d = P.shape[1]
    out = {"P": P, "eps": np.float64(case["eps"]), "nu": np.int64(case["nu"]),
           "force_general": np.int64(case.get("force_general", False)), "kernel": np.array(case["kernel"])}
    if Q is not None:
        out["Q"] = np.ascontiguousarray(Q, dtype=np.float64)
    cloud = PointCloud.from_points(P, Q)
    try:
        tree = build_tree(cloud, nu=case["nu"], eta=float(np.sqrt(2.0)))
    except ValueError as exc:
        out["error"] = np.array(str(exc))
        return out
    out.update(export_tree(tree, d))
    if case["kernel"] in ("laplace-3d", "log", "gaussian-scaled"):
        kern = custom_kernel(h, case["kernel"], d)
    else:
        kern = builtin_kernel(case["kernel"], d)
    H = assemble(tree, kern, case["eps"], force_general=bool(case.get("force_general", False)))
    out.update(export_h2(H, tree))
    nrhs = case.get("nrhs", 1)
    rng = np.random.default_rng(rng_seed)
    W = rng.standard_normal((cloud.n_sources, nrhs))
    U = np.stack([h2_matvec(H, W[:, r]) for r in range(nrhs)], axis=1)
    Ud = np.stack([dense_matvec(kern, cloud, W[:, r]) for r in range(nrhs)], axis=1)
    out["W"], out["U"], out["U_dense"] = W, U, Ud
    return out


def aca_goldens(h):
    from h2cross._accel import _core

    rng = np.random.default_rng(21)
    out = {}
    specs = [(2, 1e-4, 3, 80, 120, 1e-8), (3, 1e-4, 2, 60, 60, 1e-10), (4, 1e-4, 3, 150, 40, 1e-6),
             (0, 1e-4, 2, 100, 90, 1e-9), (1, 1e-4, 2, 70, 200, 1e-7), (2, 1e-4, 3, 5, 300, 1e-12)]
    for n, (kind, a, d, m, nn, eps) in enumerate(specs):
        X = rng.uniform(-0.5, 0.5, (m, d))
        Y = rng.uniform(-0.5, 0.5, (nn, d)) + 2.5
        U, V, rp, cp, conv, nev = _core.aca_kernel(kind, a, X, Y, eps, min(m, nn))
        out.update({f"A{n}_kind": np.int64(kind), f"A{n}_a": np.float64(a), f"A{n}_eps": np.float64(eps),
                    f"A{n}_X": X, f"A{n}_Y": Y, f"A{n}_U": U, f"A{n}_V": V, f"A{n}_rp": rp, f"A{n}_cp": cp,
                    f"A{n}_conv": np.int64(conv), f"A{n}_nevals": np.int64(nev)})
    # admissibility on boxes near the 2D tie (one-axis gap of one cell)
    from h2cross.geometry import boxes_admissible

    cx, hw, res = [], [], []
    for _ in range(4000):
        d = int(rng.integers(2, 5))
        level = int(rng.integers(2, 9))
        half = float(rng.uniform(0.5, 2.0)) * (1 + 1e-12)
        lo0 = rng.uniform(-1, 1, d) - half
        width = half * 2.0 ** (1 - level)
        mi = rng.integers(0, 1 << level, d)
        off = rng.integers(-3, 4, d)
        mj = np.clip(mi + off, 0, (1 << level) - 1)
        ca = lo0 + (mi.astype(np.float64) + 0.5) * width
        cb = lo0 + (mj.astype(np.float64) + 0.5) * width
        pad = np.zeros(4)
        pa, pb = pad.copy(), pad.copy()
        pa[:d], pb[:d] = ca, cb
        cx.append(np.concatenate([[d], pa, pb]))
        hw.append(0.5 * width)
        res.append(boxes_admissible(ca, 0.5 * width, cb, 0.5 * width, float(np.sqrt(2.0))))
    out["adm_c"] = np.array(cx)
    out["adm_hw"] = np.array(hw)
    out["adm_res"] = np.array(res, dtype=np.int64)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    h = build_reference(args.ref)
    for case in CASES:
        if args.only and case["name"] != args.only:
            continue
        out = run_case(h, case)
        np.savez_compressed(os.path.join(HERE, f"{case['name']}.npz"), **out)
        print("wrote", case["name"], "depth", out.get("depth"), out.get("error", ""))
    if not args.only:
        np.savez_compressed(os.path.join(HERE, "aca_blocks.npz"), **aca_goldens(h))
        print("wrote aca_blocks")


if __name__ == "__main__":
    main()
