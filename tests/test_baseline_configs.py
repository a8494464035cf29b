"""Parity at every BASELINE.json config, at the config's stated N (GPU vs the CPU oracle).

For c0..c4 (bench.CONFIGS, BASELINE.json "configs"), on the config's own seeded
inputs, this asserts what north_star asks of the product path:

  * tree partition, leaf membership, neighbour and interaction lists
    bit-exact against the oracle's restatement of geometry.py:230-345
    (build_tree / _annotate_level), every level;
  * every pivot index set (t_in, s_in, t_out, s_out) identical to the
    oracle's select_pivots (compress.py:216-282, _core.pyx:70-191), every
    cell of every level, and the entry-evaluation counts equal;
  * the H2 matvec within relative L2 1e-10 of the oracle's FP64 H2 matvec
    (matvec.py:142-166), every right-hand side;
  * on 1000 sampled rows, the error against a direct dense sum equal to the
    oracle's own (the NNCA approximation error of the reference algorithm;
    BASELINE tolerance vs that error is reported, not asserted: the
    reference misses it on c3).

The oracle (C, OpenMP) is the slow part: c4 (N = 4,194,304) and c1 dominate.
"""

import os
import sys
import time

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

pytestmark = pytest.mark.gpu

TREE_FIELDS = ("key", "t_ptr", "t_idx", "s_ptr", "s_idx", "nb_ptr", "nb_idx", "il_ptr", "il_idx")
PIVOT_FIELDS = ("k_in", "k_out", "t_in", "s_in", "t_out", "s_out")


@pytest.fixture(scope="module")
def h2c():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_14832_b200 as h2c

    return h2c


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3", "c4"])
def test_baseline_config_parity(h2c, oracle_mod, name):
    import bench

    cfg = bench.CONFIGS[name]
    dist, n, dim, seed, kname, kkw, nu, eps, xdist, nrhs = cfg
    pts, w = bench.make_inputs(cfg)
    kern = h2c.builtin_kernel(kname, dim, **kkw)
    eta = float(np.sqrt(2.0))
    t0 = time.perf_counter()
    cloud = h2c.PointCloud.from_points(pts)
    tree = h2c.build_tree(cloud, nu=nu, eta=eta)
    h2 = h2c.assemble(tree, kern, eps)
    t_gpu = time.perf_counter() - t0

    t0 = time.perf_counter()
    ot = oracle_mod.OTree(pts, None, nu=nu, eta=eta)
    oh = oracle_mod.OH2(ot, kern.kind, kern.device_param, eps)
    t_orc = time.perf_counter() - t0

    # tree and lists: bit-exact
    assert tree.depth == ot.depth and tree.over_capacity == ot.over_capacity
    for level in range(tree.depth + 1):
        for f in TREE_FIELDS:
            assert np.array_equal(tree.array(level, f), ot.get(level, f)), (name, level, f)
    # pivots: every set identical, same entry-evaluation counts
    for level in range(2, tree.depth + 1):
        for f in PIVOT_FIELDS:
            assert np.array_equal(h2.array(level, f), oh.get(level, f)), (name, level, f)
    st = oh.stats()
    assert h2.stats.evals_pivots == st["evals_pivots"]
    assert h2.stats.evals_couplings == st["evals_couplings"]
    assert h2.stats.evals_nearfield == st["evals_nearfield"]
    assert h2.stats.max_rank == st["max_rank"]

    # matvec vs the oracle's FP64 H2 matvec
    u = h2c.h2_matvec(h2, w)
    uo = oh.matvec(w)
    err = float(np.linalg.norm(u - uo) / np.linalg.norm(uo))
    assert err <= 1e-10, (name, err)

    # approximation error on 1000 sampled rows: GPU and oracle carry the same NNCA error
    rows = np.random.default_rng(7).choice(n, 1000, replace=False)
    w0 = w if w.ndim == 1 else w[:, 0]
    u0 = u if u.ndim == 1 else u[:, 0]
    uo0 = uo if uo.ndim == 1 else uo[:, 0]
    exact = oracle_mod.dense_rows(kern.kind, kern.device_param, pts, rows, pts, w0)
    exact_gpu = h2c.dense_rows(kern, cloud, rows, w0)
    assert np.allclose(exact_gpu, exact, rtol=1e-12, atol=1e-12 * np.abs(exact).max())
    e_gpu = float(np.linalg.norm(u0[rows] - exact) / np.linalg.norm(exact))
    e_orc = float(np.linalg.norm(uo0[rows] - exact) / np.linalg.norm(exact))
    assert abs(e_gpu - e_orc) <= 1e-6 * e_orc + 1e-13, (e_gpu, e_orc)
    print(f"\n[{name}] N={n} depth={tree.depth} gpu setup {t_gpu:.2f}s oracle setup {t_orc:.2f}s "
          f"rel_l2_vs_oracle_h2={err:.2e} dense1000 gpu={e_gpu:.3e} oracle={e_orc:.3e} eps={eps:g} "
          f"eps_ratio={e_gpu / eps:.2f}")
