"""GPU tests of the drop-in API around the hot path: coefficient collection (matvec.py:169 collect=True),
scratch reuse across right-hand-side widths, stream discipline of the C ABI, argument checks, pinned buffers."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h2c():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_14832_b200 as h2c

    return h2c


def close(a, b, tol=1e-12):
    """Equal up to the summation order of the symmetric kernel's FP64 reductions (atomics: not bitwise repeatable)."""
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and float(np.abs(a - b).max()) <= tol * float(np.abs(b).max())


@pytest.fixture(scope="module")
def problem(h2c):
    from paper_2203_14832_b200 import sampling

    pts = sampling.sphere_points(6000, 3, 2)
    cloud = h2c.PointCloud.from_points(pts)
    tree = h2c.build_tree(cloud, nu=64, eta=float(np.sqrt(2.0)))
    kern = h2c.builtin_kernel("laplace-3d", 3)
    h2 = h2c.assemble(tree, kern, 1e-8)
    return cloud, tree, kern, h2


def test_collect_coefficients(h2c, problem):
    """w_out of a leaf = p2m^T w[s_idx]; u on a leaf = l2p u_in + near field (the reference's pass 1 and pass 5)."""
    cloud, tree, kern, h2 = problem
    w = np.random.default_rng(3).standard_normal(cloud.n_sources)
    u, coeffs = h2c.h2_matvec_reference(h2, w, collect=True)
    assert close(u, h2c.h2_matvec(h2, w))
    cells = {c for level in h2.compressed_levels() for c in tree.nonempty_cells(level)}
    assert set(coeffs) == cells
    checked = 0
    for cell in tree.nonempty_cells(tree.depth)[:40]:
        w_out, u_in = coeffs[cell]
        ps = h2.pivot_set(cell)
        assert w_out.shape == (ps.s_out.size,) and u_in.shape == (ps.t_in.size,)
        ops = h2.transfers[cell]
        ref = ops.p2m.T @ w[cell.s_idx]
        assert np.allclose(w_out, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        near = np.zeros(cell.t_idx.size)
        for y in cell.neighbors:
            if y.s_idx.size:
                near += h2.nearfield[(cell, y)] @ w[y.s_idx]
        ref_u = ops.l2p @ u_in + near
        assert np.allclose(u[cell.t_idx], ref_u, rtol=1e-10, atol=1e-10 * np.abs(ref_u).max())
        checked += 1
    assert checked == 40
    # an upper level: w_out = sum over children of m2m w_out(child)  (pass 2)
    level = tree.depth - 1
    for cell in tree.nonempty_cells(level)[:10]:
        ops = h2.transfers[cell]
        acc = np.zeros(h2.pivot_set(cell).s_out.size)
        for child, mat in ops.m2m.items():
            acc += mat @ coeffs[child][0]
        assert np.allclose(coeffs[cell][0], acc, rtol=1e-11, atol=1e-12 * max(np.abs(acc).max(), 1e-300))


def test_collect_needs_single_vector(h2c, problem):
    cloud, tree, kern, h2 = problem
    with pytest.raises(ValueError):
        h2c.h2_matvec_reference(h2, np.ones((cloud.n_sources, 2)), collect=True)


def test_alternating_rhs_widths(h2c, problem):
    """Scratch sets of several widths are kept side by side: alternating widths returns the same numbers."""
    cloud, tree, kern, h2 = problem
    rng = np.random.default_rng(5)
    W = rng.standard_normal((cloud.n_sources, 17))
    u1 = h2c.h2_matvec(h2, W[:, 0].copy())
    U17 = h2c.h2_matvec(h2, W)
    u1b = h2c.h2_matvec(h2, W[:, 0].copy())
    U16 = h2c.h2_matvec(h2, np.ascontiguousarray(W[:, :16]))
    U17b = h2c.h2_matvec(h2, W)
    U3 = h2c.h2_matvec(h2, np.ascontiguousarray(W[:, :3]))
    u1c = h2c.h2_matvec(h2, W[:, 0].copy())
    assert close(u1, u1b) and close(u1, u1c)
    assert close(U17, U17b)
    scale = np.abs(u1).max()
    assert np.abs(U17[:, 0] - u1).max() <= 1e-11 * scale
    assert np.abs(U16 - U17[:, :16]).max() <= 1e-11 * scale
    assert np.abs(U3 - U17[:, :3]).max() <= 1e-11 * scale


def test_two_streams_one_matrix(h2c, problem):
    """Products on different streams of one matrix are ordered by the handle's event: no scratch race."""
    import torch

    cloud, tree, kern, h2 = problem
    rng = np.random.default_rng(7)
    ws = [torch.from_numpy(rng.standard_normal(cloud.n_sources)).cuda() for _ in range(6)]
    ref = [h2c.h2_matvec(h2, w).clone() for w in ws]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i, w in enumerate(ws):
        with torch.cuda.stream(streams[i % 2]):
            outs.append(h2c.h2_matvec(h2, w))
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert close(a.cpu().numpy(), b.cpu().numpy())


def test_free_while_product_in_flight(h2c):
    """Dropping the matrix right after launching on a side stream is safe (the free waits for the handle's event)."""
    import torch
    from paper_2203_14832_b200 import sampling

    pts = sampling.sphere_points(4000, 3, 9)
    cloud = h2c.PointCloud.from_points(pts)
    tree = h2c.build_tree(cloud, nu=64, eta=float(np.sqrt(2.0)))
    kern = h2c.builtin_kernel("laplace-3d", 3)
    w = torch.from_numpy(np.random.default_rng(1).standard_normal(4000)).cuda()
    h2 = h2c.assemble(tree, kern, 1e-6)
    ref = h2c.h2_matvec(h2, w).clone()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        out = h2c.h2_matvec(h2, w)
    del h2
    import gc

    gc.collect()
    h2b = h2c.assemble(tree, kern, 1e-6)  # reuses the pool's memory
    again = h2c.h2_matvec(h2b, w)
    torch.cuda.synchronize()
    assert close(out.cpu().numpy(), ref.cpu().numpy()) and close(again.cpu().numpy(), ref.cpu().numpy())


def test_dense_rows_range_check(h2c, problem):
    cloud, tree, kern, h2 = problem
    w = np.ones(cloud.n_sources)
    with pytest.raises(IndexError):
        h2c.dense_rows(kern, cloud, np.array([0, cloud.n_targets]), w)
    with pytest.raises(IndexError):
        h2c.dense_rows(kern, cloud, np.array([-1]), w)
    rows = np.array([0, 5, cloud.n_targets - 1])
    full = h2c.dense_matvec(kern, cloud, w)
    assert np.allclose(h2c.dense_rows(kern, cloud, rows, w), full[rows], rtol=1e-13)


def test_pinned_buffers(h2c, problem):
    cloud, tree, kern, h2 = problem
    w = h2c.pinned_empty(cloud.n_sources)
    assert w.shape == (cloud.n_sources,) and w.dtype == np.float64
    w[:] = np.random.default_rng(11).standard_normal(cloud.n_sources)
    out = h2c.pinned_empty(cloud.n_targets)
    u = h2c.h2_matvec(h2, w, out=out)
    assert u is out
    assert close(u, h2c.h2_matvec(h2, np.array(w)))
    W = h2c.pinned_empty((cloud.n_sources, 2))
    assert W.shape == (cloud.n_sources, 2) and W.flags.c_contiguous


def test_release_workspace_then_assemble(h2c, problem):
    cloud, tree, kern, h2 = problem
    before = h2.array(tree.depth, "t_in").copy()
    h2c.release_workspace()
    h2b = h2c.assemble(tree, kern, 1e-8)
    assert np.array_equal(h2b.array(tree.depth, "t_in"), before)


def test_reference_memory_bytes(h2c, problem):
    cloud, tree, kern, h2 = problem
    st = h2.stats
    ref = h2.reference_memory_bytes()
    assert ref > 8 * (st.evals_couplings + st.evals_nearfield)
    # spot check against the views: one leaf's blocks
    cell = tree.nonempty_cells(tree.depth)[0]
    ops = h2.transfers[cell]
    assert ops.l2p.nbytes == 8 * cell.t_idx.size * h2.pivot_set(cell).t_in.size
    assert h2.memory_bytes() > 0


def test_setup_is_bitwise_repeatable(h2c):
    """The ACA kernel's work queue, prefetch ring and reductions are timing-dependent machinery; the pivots,
    ranks, evaluation counts and interpolators it exports are not."""
    from paper_2203_14832_b200 import sampling

    pts = sampling.sphere_points(20000, 3, 5)
    cloud = h2c.PointCloud.from_points(pts)
    tree = h2c.build_tree(cloud, nu=64, eta=float(np.sqrt(2.0)))
    kern = h2c.builtin_kernel("laplace-3d", 3)
    runs = []
    for _ in range(3):
        h2 = h2c.assemble(tree, kern, 1e-8)
        arrays = {(level, f): h2.array(level, f).copy() for level in h2.compressed_levels()
                  for f in ("k_in", "t_in", "s_in", "nevals", "converged")}
        cell = tree.nonempty_cells(tree.depth - 1)[3]
        runs.append((arrays, h2.interp(cell.level, cell._ref_index, 0)))
    for arrays, P in runs[1:]:
        assert all(np.array_equal(arrays[k], runs[0][0][k]) for k in arrays)
        assert np.array_equal(P, runs[0][1])
