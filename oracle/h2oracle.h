/*
 * h2oracle — CPU restatement of the reference h2cross hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2203_14832_b200/ links, loads
 * or calls this library.  It is used by tests/ (as the parity checker), by
 * __graft_entry__.smoke() (as the checker) and by bench.py's cpu_baseline /
 * --impl reference legs (as the timed CPU implementation of the reference
 * algorithm).  Each function cites the reference file:line it restates
 * (paths relative to /root/reference/pkg/src/h2cross/).
 *
 * Pinning: golden vectors produced by the reference package itself
 * (tests/golden/make_golden.py) are compared against this oracle in
 * tests/test_oracle_golden.py — tree membership, lists and pivot sets
 * bit-exact, matvec outputs to 1e-12.
 */
#ifndef H2ORACLE_H
#define H2ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oh2_tree oh2_tree;
typedef struct oh2_h2 oh2_h2;

/* kernels.py:28-33 kind ids, plus the B200 additions (5..7) */
enum {
  OH2_REG_LOG = 0, OH2_REG_INVERSE = 1, OH2_COULOMB = 2, OH2_MATERN = 3,
  OH2_GAUSSIAN = 4, OH2_LAPLACE = 5, OH2_LOG = 6, OH2_GAUSSIAN_SCALED = 7
};

const char* oh2_last_error(void);
void oh2_set_threads(int n);
int oh2_get_threads(void);

/* geometry.py:230 build_tree (+ geometry.py:322 _annotate_level) */
int oh2_build_tree(const double* P, int64_t np, const double* Q, int64_t nq, int d,
                   int shared, int64_t nu, double eta, oh2_tree** out);
void oh2_tree_free(oh2_tree* t);
int oh2_tree_depth(const oh2_tree* t);
int oh2_tree_over_capacity(const oh2_tree* t);
void oh2_tree_root(const oh2_tree* t, double* mid, double* half);
int64_t oh2_tree_ncells(const oh2_tree* t, int level);
/* what: 0 key(n) 1 mi(n*d) 2 t_ptr(n+1) 3 t_idx 4 s_ptr(n+1) 5 s_idx
 *       6 nb_ptr(n+1) 7 nb_idx 8 il_ptr(n+1) 9 il_idx 10 parent(n)
 *       11 ch_ptr(n+1) 12 ch_idx ; returns element count, copies if dst */
int64_t oh2_tree_get(const oh2_tree* t, int level, int what, int64_t* dst);

/* geometry.py:147 boxes_admissible */
int oh2_boxes_admissible(const double* cx, double hwx, const double* cy, double hwy, int d, double eta);

/* _core.pyx:15 _kval + :38 _r2 ; _core.pyx:47 kernel_block */
double oh2_kval(int kind, double a, double r2);
void oh2_kernel_block(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n,
                      int d, double* out);

/* _core.pyx:70 aca_kernel.  U (m x k) and V (n x k) row-major, rp/cp local
 * pivots.  Buffers must hold cap columns.  Returns rank k. */
int64_t oh2_aca(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d,
                double eps, int64_t cap, double* U, double* V, int64_t* rp, int64_t* cp,
                int* converged, int64_t* nevals);

/* aca.py:297 row_interpolator / aca.py:311 col_interpolator on factors from
 * oh2_aca (row-major m x k / n x k).  out: row-major (rows x k). */
void oh2_row_interpolator(const double* U, int64_t m, int64_t k, const int64_t* rp, double* out);
void oh2_col_interpolator(const double* V, int64_t n, int64_t k, const int64_t* cp, double* out);

/* compress.py:285 assemble / :216 select_pivots.  max_rank < 0 means None */
int oh2_assemble(const oh2_tree* t, int kind, double a, double eps, int force_general,
                 int64_t max_rank, oh2_h2** out);
void oh2_h2_free(oh2_h2* h);
/* per (level, cell) exports.  what: 0 k_in(n) 1 k_out(n) 2 t_in(ptr by k_in)
 * 3 s_in 4 t_out(ptr by k_out) 5 s_out 6 nevals(n) 7 converged_in(n) */
int64_t oh2_h2_get_i64(const oh2_h2* h, int level, int what, int64_t* dst);
/* interpolation operator of one cell: which 0 = row interp (l2p / stacked
 * l2l, m_in x k_in), 1 = col interp (p2m / stacked m2m^T, n_out x k_out).
 * Returns rows; copies row-major if dst. */
int64_t oh2_h2_get_interp(const oh2_h2* h, int level, int64_t cell, int which, int64_t* cols,
                          double* dst);
void oh2_h2_stats(const oh2_h2* h, int64_t* evals_pivots, int64_t* evals_couplings,
                  int64_t* evals_nearfield, int64_t* max_rank, int64_t* cells_visited);

/* matvec.py:169 h2_matvec_reference with regenerated S and near-field blocks.
 * w: n_sources x nrhs (row-major), u: n_targets x nrhs. */
int oh2_matvec(const oh2_h2* h, const double* w, double* u, int64_t nrhs);
/* matvec.py:233 dense_matvec */
void oh2_dense_matvec(int kind, double a, const double* P, int64_t np, const double* Q, int64_t nq,
                      int d, const double* w, double* u, int64_t nrhs);
void oh2_dense_rows(int kind, double a, const double* P, const int64_t* rows, int64_t nrows,
                    const double* Q, int64_t nq, int d, const double* w, double* u);

#ifdef __cplusplus
}
#endif
#endif
