/*
 * h2b.h — C ABI of libh2b200.so, the B200-native NNCA / H2 matvec engine.
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures
 * (streams are passed as opaque void*, 0 = the legacy default stream).
 * Every function returns 0 on success and a negative code on failure, with
 * the message in h2b_last_error().  Point arrays are row-major (n, d)
 * float64, exactly as the reference's numpy arrays.  Pointer arguments are
 * host memory unless the call takes `on_device` and it is nonzero.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to h2cross/ in the reference package).
 */
#ifndef H2B_H
#define H2B_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct h2b_tree h2b_tree;
typedef struct h2b_h2 h2b_h2;

/* kernel kinds: kernels.py:28-33 (0..4) plus B200 additions */
enum {
  H2B_REG_LOG = 0,         /* reg-log-2d, param a = reg_a */
  H2B_REG_INVERSE = 1,     /* reg-inverse, param a = reg_a */
  H2B_COULOMB = 2,         /* 1/r, K(x,x)=0 */
  H2B_MATERN = 3,          /* exp(-r) */
  H2B_GAUSSIAN = 4,        /* exp(-r^2) */
  H2B_LAPLACE = 5,         /* 1/(4 pi r), K(x,x)=0 */
  H2B_LOG = 6,             /* log r, K(x,x)=0 */
  H2B_GAUSSIAN_SCALED = 7  /* exp(-a r^2) */
};

const char* h2b_last_error(void);
int h2b_version(void);

/* ---- fused kernel evaluation: _accel/_core.pyx:47 kernel_block ---- */
int h2b_kernel_block(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d,
                     double* out);
/* _accel/_core.pyx:59 kernel_row */
int h2b_kernel_row(int kind, double a, const double* x, const double* Y, int64_t n, int d, double* out);
/* _accel/_core.pyx:70 aca_kernel: partially pivoted ACA on K(X_i, Y_j).
 * U (m x cap) and V (n x cap) row-major, first *rank columns valid;
 * rp / cp: local pivots in discovery order. */
int h2b_aca_kernel(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d,
                   double eps, int64_t cap, double* U, double* V, int64_t* rp, int64_t* cp, int* converged,
                   int64_t* nevals, int64_t* rank);

/* ---- tree: geometry.py:230 build_tree (+ :339 compute_lists) ---- */
int h2b_tree_build(const double* P, int64_t np, const double* Q, int64_t nq, int d, int shared, int64_t nu,
                   double eta, int on_device, void* stream, h2b_tree** out);
void h2b_tree_free(h2b_tree* t);
/* depth, over_capacity flag, root box (mid[d], half) */
int h2b_tree_info(const h2b_tree* t, int* depth, int* over_capacity, double* mid, double* half);
/* number of nonempty cells at a level */
int64_t h2b_tree_ncells(const h2b_tree* t, int level);
/* Per-level arrays in the reference's cell order (nonempty cells sorted by
 * multi-index, geometry.py:175).  what: 0 key 1 multi_index(n*d) 2 t_ptr
 * 3 t_idx 4 s_ptr 5 s_idx 6 nb_ptr 7 nb_idx 8 il_ptr 9 il_idx 10 parent
 * 11 ch_ptr 12 ch_idx.  Returns the element count; copies when dst != 0. */
int64_t h2b_tree_get(const h2b_tree* t, int level, int what, int64_t* dst);

/* ---- NNCA assembly: compress.py:285 assemble / :216 select_pivots ---- */
/* max_rank < 0 means None (cap = min(rows, cols)). */
int h2b_assemble(const h2b_tree* t, int kind, double a, double eps, int force_general, int64_t max_rank,
                 void* stream, h2b_h2** out);
/* Both free functions first wait for the last work submitted on the handle (any stream).  Free every H2 built
 * on a tree before the tree. */
void h2b_h2_free(h2b_h2* h);
/* Releases the per-device ACA workspace arenas kept between assemblies (tens of GB after a large setup). */
int h2b_release_workspace(void);
/* per level (>= 2), reference cell order.  what: 0 k_in 1 k_out 2 t_in
 * 3 s_in 4 t_out 5 s_out 6 nevals 7 converged(in) 8 m_in(rows of the row
 * interpolator) 9 n_out(rows of the column interpolator) */
int64_t h2b_h2_get_i64(const h2b_h2* h, int level, int what, int64_t* dst);
/* interpolation operator of one cell (reference order index): which 0 =
 * row interpolator (l2p for leaves, stacked l2l blocks otherwise), 1 =
 * column interpolator (p2m / stacked m2m^T).  Row-major copy to dst. */
int64_t h2b_h2_get_interp(const h2b_h2* h, int level, int64_t cell, int which, int64_t* cols, double* dst);
/* Coefficient vectors of the last single-vector product (matvec.py:169 h2_matvec_reference(collect=True)):
 * which 0 = w_out (outgoing, after P2M / M2M), 1 = u_in (incoming, after M2L and L2L), cells concatenated in the
 * reference order, k_out / k_in entries per cell.  Returns the element count; copies when dst != 0. */
int64_t h2b_h2_get_coeffs(h2b_h2* h, int level, int which, double* dst);
/* stats[0..9]: evals_pivots evals_couplings evals_nearfield max_rank
 * cells_visited memory_bytes symmetric setup_ns depth aca_unconverged */
int h2b_h2_stats(const h2b_h2* h, int64_t* stats);

/* ---- matvec: matvec.py:142 h2_matvec ---- */
/* w: (n_sources, nrhs) row-major, u: (n_targets, nrhs). */
/* The product uses scratch owned by h: concurrent callers on one h are serialised (host mutex), and a call on a
 * stream other than the previous one first waits (cudaStreamWaitEvent) for the previous call's work.  Scratch
 * sets of up to four right-hand-side widths are kept, so alternating nrhs does not rebuild them. */
int h2b_matvec(h2b_h2* h, const double* w, double* u, int64_t nrhs, int on_device, void* stream);
/* Page-locked host memory for w / u of the host-pointer calls (on_device = 0). */
int h2b_host_alloc(void** p, int64_t bytes);
void h2b_host_free(void* p);
/* Number of kernel launches one h2b_matvec call issues (for bench accounting). */
int64_t h2b_matvec_launches(const h2b_h2* h, int64_t nrhs);
/* Per-stage device times (ms) of the last profiled matvec: [p2m+m2m, m2l, l2l, p2p+l2p, total];
 * enable with h2b_set_profiling(1). */
int h2b_set_profiling(int on);
int h2b_last_stage_ms(double* ms5);
/* Measured FP64 FMA throughput of this device (TFLOP/s), the roofline
 * denominator for the FP64-bound interaction kernels. */
int h2b_fp64_peak(double* tflops);

/* ---- dense oracles: matvec.py:233 dense_matvec / :245 dense_rows ---- */
int h2b_dense_matvec(int kind, double a, const double* P, int64_t np, const double* Q, int64_t nq, int d,
                     const double* w, double* u, int64_t nrhs, int on_device, void* stream);
/* rows[i] must lie in [0, np) (ValueError otherwise; the reference raises IndexError) */
int h2b_dense_rows(int kind, double a, const double* P, int64_t np, const int64_t* rows, int64_t nrows,
                   const double* Q, int64_t nq, int d, const double* w, double* u);

#ifdef __cplusplus
}
#endif
#endif
