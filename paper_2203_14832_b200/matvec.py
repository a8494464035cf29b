"""H2 matrix-vector product, dense oracle and error metrics (matvec.py of h2cross).

``h2_matvec`` runs the level-batched GPU product (h2b_matvec): P2M, M2M,
M2L at every level with the coupling entries regenerated in registers, L2L,
and one fused near-field + L2P kernel that writes the result in the caller's
point order.  Accepts numpy arrays (host in / host out, copies included) or
float64 CUDA torch tensors (device-resident, zero copy, runs on the current
torch stream).  ``w`` may be (n,) as in the reference or (n, nrhs).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .compress import H2Matrix
from .kernels import KernelSpec


def _is_torch_cuda(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch") and getattr(x, "is_cuda", False)


def h2_matvec(h2: H2Matrix, w):
    """Apply the compressed operator: u = A w (matvec.py:483)."""
    n_t, n_s = h2.shape
    L = _lib.lib()
    if _is_torch_cuda(w):
        import torch

        if w.dtype != torch.float64:
            raise ValueError("device vectors must be float64")
        if w.shape[0] != n_s or w.dim() not in (1, 2):
            raise ValueError(f"vector has shape {tuple(w.shape)}, expected ({n_s},) or ({n_s}, nrhs)")
        w = w.contiguous()
        nrhs = 1 if w.dim() == 1 else w.shape[1]
        u = torch.empty((n_t,) if w.dim() == 1 else (n_t, nrhs), dtype=torch.float64, device=w.device)
        stream = torch.cuda.current_stream(w.device).cuda_stream
        _lib.check(L.h2b_matvec(h2.handle, w.data_ptr(), u.data_ptr(), nrhs, 1, stream))
        return u
    w = np.asarray(w, dtype=np.float64)
    if w.ndim not in (1, 2) or w.shape[0] != n_s:
        raise ValueError(f"vector has shape {w.shape}, expected ({n_s},)")
    w = np.ascontiguousarray(w)
    nrhs = 1 if w.ndim == 1 else w.shape[1]
    u = np.empty((n_t,) if w.ndim == 1 else (n_t, nrhs))
    _lib.check(L.h2b_matvec(h2.handle, w.ctypes.data, u.ctypes.data, nrhs, 0, None))
    return u


def h2_matvec_reference(h2: H2Matrix, w, collect: bool = False):
    """matvec.py:510 — the engine has a single (device) product; ``collect`` is unsupported."""
    if collect:
        raise NotImplementedError("per-cell coefficient collection is not exposed by the B200 engine")
    return h2_matvec(h2, w)


def dense_matvec(kernel: KernelSpec, cloud, w):
    """Exact O(N^2) product by direct evaluation on the GPU (matvec.py:574)."""
    kernel.require_device()
    w = np.asarray(w, dtype=np.float64)
    if w.shape[0] != cloud.n_sources or w.ndim not in (1, 2):
        raise ValueError(f"vector has shape {w.shape}, expected ({cloud.n_sources},)")
    w = np.ascontiguousarray(w)
    nrhs = 1 if w.ndim == 1 else w.shape[1]
    u = np.empty((cloud.n_targets,) if w.ndim == 1 else (cloud.n_targets, nrhs))
    P, Q = cloud.points_p, cloud.points_q
    _lib.check(_lib.lib().h2b_dense_matvec(kernel.kind, kernel.device_param, P.ctypes.data, P.shape[0],
                                           Q.ctypes.data, Q.shape[0], P.shape[1], w.ctypes.data, u.ctypes.data,
                                           nrhs, 0, None))
    return u


def dense_rows(kernel: KernelSpec, cloud, rows, w) -> np.ndarray:
    """Exact values of selected output rows (matvec.py:586), on the GPU."""
    kernel.require_device()
    rows = _lib.i64(rows)
    w = _lib.f64(w)
    u = np.empty(rows.size)
    P, Q = cloud.points_p, cloud.points_q
    _lib.check(_lib.lib().h2b_dense_rows(kernel.kind, kernel.device_param, _lib.dptr(P), _lib.iptr(rows), rows.size,
                                         _lib.dptr(Q), Q.shape[0], P.shape[1], _lib.dptr(w), _lib.dptr(u)))
    return u


def relative_error(u, u_ref) -> float:
    """||u - u_ref||_2 / ||u_ref||_2 (matvec.py:592)."""
    u = np.asarray(u, dtype=np.float64)
    u_ref = np.asarray(u_ref, dtype=np.float64)
    if u.shape != u_ref.shape:
        raise ValueError("length mismatch")
    ref = float(np.linalg.norm(u_ref))
    if ref == 0.0:
        raise ValueError("zero reference vector")
    return float(np.linalg.norm(u - u_ref)) / ref


def matvec_launches(h2: H2Matrix, nrhs: int = 1) -> int:
    """Number of kernel launches one product issues."""
    return int(_lib.lib().h2b_matvec_launches(h2.handle, int(nrhs)))


def stage_times(h2: H2Matrix, w, repeats: int = 3):
    """Per-stage device times (ms) [upward, M2L, L2L, near+L2P, total] of a product."""
    import ctypes

    L = _lib.lib()
    L.h2b_set_profiling(1)
    try:
        for _ in range(repeats):
            h2_matvec(h2, w)
        out = np.zeros(5)
        L.h2b_last_stage_ms(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return out
    finally:
        L.h2b_set_profiling(0)
