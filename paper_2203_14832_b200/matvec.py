"""H2 matrix-vector product, dense oracle and error metrics (matvec.py of h2cross).

``h2_matvec`` runs the level-batched GPU product (h2b_matvec): P2M, M2M,
M2L at every level and the near field with the coupling entries regenerated
in registers (on the symmetric path each unordered cell pair once, applied
both ways), L2L, and L2P, writing the result in the caller's point order.
Accepts numpy arrays, CPU torch tensors (pinned: asynchronous copies) or
float64 CUDA torch tensors (device-resident, zero copy, current torch
stream).  ``w`` may be (n,) as in the reference or (n, nrhs).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .compress import H2Matrix
from .kernels import KernelSpec


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def h2_matvec(h2: H2Matrix, w, out=None):
    """Apply the compressed operator: u = A w (matvec.py:142).

    ``w`` is (n,) as in the reference or (n, nrhs); float64.  Accepted forms:

    * numpy array: host in / host out (the copies go through the driver's staging);
    * CPU torch tensor, ideally pinned (``pin_memory()``): host in / host out with asynchronous copies on the
      current CUDA stream -- the end-to-end path ``bench.py`` times;
    * CUDA torch tensor: device-resident, zero copy, on the current torch stream.

    ``out`` (same kind and shape as the result) avoids allocating the result on every call.
    """
    n_t, n_s = h2.shape
    L = _lib.lib()
    if _is_torch(w):
        import torch

        if w.dtype != torch.float64:
            raise ValueError("vectors must be float64")
        if w.dim() not in (1, 2) or w.shape[0] != n_s:
            raise ValueError(f"vector has shape {tuple(w.shape)}, expected ({n_s},) or ({n_s}, nrhs)")
        w = w.contiguous()
        nrhs = 1 if w.dim() == 1 else w.shape[1]
        shape = (n_t,) if w.dim() == 1 else (n_t, nrhs)
        if out is None:
            out = torch.empty(shape, dtype=torch.float64, device=w.device, pin_memory=bool(not w.is_cuda
                                                                                            and w.is_pinned()))
        elif tuple(out.shape) != shape or out.dtype != torch.float64 or out.device != w.device or \
                not out.is_contiguous():
            raise ValueError(f"out must be a contiguous float64 tensor of shape {shape} on {w.device}")
        dev = w.device if w.is_cuda else torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(L.h2b_matvec(h2.handle, w.data_ptr(), out.data_ptr(), nrhs, 1 if w.is_cuda else 0, stream))
        return out
    w = np.asarray(w, dtype=np.float64)
    if w.ndim not in (1, 2) or w.shape[0] != n_s:
        raise ValueError(f"vector has shape {w.shape}, expected ({n_s},)")
    w = np.ascontiguousarray(w)
    nrhs = 1 if w.ndim == 1 else w.shape[1]
    shape = (n_t,) if w.ndim == 1 else (n_t, nrhs)
    if out is None:
        out = np.empty(shape)
    elif out.shape != shape or out.dtype != np.float64 or not out.flags.c_contiguous:
        raise ValueError(f"out must be a C-contiguous float64 array of shape {shape}")
    _lib.check(L.h2b_matvec(h2.handle, w.ctypes.data, out.ctypes.data, nrhs, 0, None))
    return out


def h2_matvec_reference(h2: H2Matrix, w, collect: bool = False):
    """matvec.py:169 -- the engine has a single (device) product.

    With ``collect=True`` also returns {cell: (w_out, u_in)}, the per-cell outgoing / incoming coefficient
    vectors of this product, read back from the device (the level buffers of the upward pass and of M2L + L2L).
    """
    u = h2_matvec(h2, w)
    if not collect:
        return u
    if np.ndim(u) != 1:
        raise ValueError("collect=True needs a single vector")
    L = _lib.lib()
    coeffs = {}
    for level in h2.compressed_levels():
        got = []
        for which in (0, 1):
            n = _lib.check(L.h2b_h2_get_coeffs(h2.handle, level, which, None))
            buf = np.empty(n)
            if n:
                _lib.check(L.h2b_h2_get_coeffs(h2.handle, level, which, _lib.dptr(buf)))
            got.append(buf)
        k_out, k_in = h2.array(level, "k_out"), h2.array(level, "k_in")
        po = np.concatenate([[0], np.cumsum(k_out)])
        pi = np.concatenate([[0], np.cumsum(k_in)])
        for cell in h2.tree.nonempty_cells(level):
            i = cell._ref_index
            coeffs[cell] = (got[0][po[i]:po[i + 1]].copy(), got[1][pi[i]:pi[i + 1]].copy())
    return u, coeffs


def dense_matvec(kernel: KernelSpec, cloud, w):
    """Exact O(N^2) product by direct evaluation on the GPU (matvec.py:233)."""
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
    """Exact values of selected output rows (matvec.py:245), on the GPU."""
    kernel.require_device()
    rows = _lib.i64(rows)
    w = _lib.f64(w)
    u = np.empty(rows.size)
    P, Q = cloud.points_p, cloud.points_q
    if rows.size and (rows.min() < 0 or rows.max() >= P.shape[0]):
        raise IndexError(f"row index out of range for {P.shape[0]} targets")  # the reference's fancy index raises
    _lib.check(_lib.lib().h2b_dense_rows(kernel.kind, kernel.device_param, _lib.dptr(P), P.shape[0], _lib.iptr(rows),
                                         rows.size, _lib.dptr(Q), Q.shape[0], P.shape[1], _lib.dptr(w),
                                         _lib.dptr(u)))
    return u


class _PinnedBlock:
    """Owner of one cudaHostAlloc block; freed when the last numpy view goes away."""

    def __init__(self, nbytes: int):
        import ctypes

        self.ptr = ctypes.c_void_p()
        _lib.check(_lib.lib().h2b_host_alloc(ctypes.byref(self.ptr), int(nbytes)))
        self.nbytes = int(nbytes)

    def __del__(self):
        try:
            _lib.lib().h2b_host_free(self.ptr)
        except Exception:  # interpreter shutdown
            pass


def pinned_empty(shape) -> np.ndarray:
    """float64 numpy array in page-locked host memory (cudaHostAlloc).

    ``h2_matvec(h2, w)`` with numpy ``w`` / ``out`` allocated here copies at the full PCIe rate and matches the
    end-to-end time quoted for pinned buffers; ordinary (pageable) numpy arrays go through the driver's staging.
    """
    import ctypes

    shape = (int(shape),) if np.isscalar(shape) else tuple(int(x) for x in shape)
    n = int(np.prod(shape, dtype=np.int64))
    block = _PinnedBlock(max(n, 1) * 8)
    buf = (ctypes.c_double * max(n, 1)).from_address(block.ptr.value)
    buf._h2b_owner = block  # the ctypes array is the numpy array's base: keeps the block alive
    return np.frombuffer(buf, dtype=np.float64, count=n).reshape(shape)


def release_workspace() -> None:
    """Free the per-device ACA workspace arenas the engine keeps between assemblies."""
    _lib.check(_lib.lib().h2b_release_workspace())


def relative_error(u, u_ref) -> float:
    """||u - u_ref||_2 / ||u_ref||_2 (matvec.py:251)."""
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
