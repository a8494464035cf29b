// matvec.cu — level-batched H2 matrix-vector product (matvec.py:483 h2_matvec,
// the five passes of matvec.py:510 h2_matvec_reference), FP64 throughout.
//
// The coupling blocks S_{X,Y} = K(t_in^X, s_out^Y) and the near-field blocks
// are NOT stored (the reference stores both): both are regenerated in
// registers inside one interaction kernel, because on B200 evaluating 1/r in
// FP64 (~12 FP64 instructions / entry) is ~3x cheaper than streaming the
// stored 8-byte entry from HBM.  Transfer operators (P2M/M2M/L2L/L2P) are
// stored dense, column-major, and applied as batched small GEMVs whose
// operands are contiguous slices thanks to the Morton cell order.
#include <cmath>

#include "engine.cuh"

namespace h2b {

namespace {

bool g_profile = false;
double g_stage_ms[5] = {0, 0, 0, 0, 0};

struct KParams {
  double a, inv_log_a, c_near;  // reg-log constants
};

// fast kernel evaluation (matvec path; tolerance 1e-10 relative)
template <int KIND>
__device__ __forceinline__ double kfast(double r2, const KParams& kp) {
  if constexpr (KIND == COULOMB || KIND == LAPLACE) {
    return r2 > 0.0 ? rsqrt(r2) : 0.0;  // LAPLACE's 1/(4 pi) applied to the sum
  } else if constexpr (KIND == GAUSSIAN) {
    return exp(-r2);
  } else if constexpr (KIND == GAUSSIAN_SCALED) {
    return exp(-kp.a * r2);
  } else if constexpr (KIND == MATERN) {
    return exp(-sqrt(r2));
  } else if constexpr (KIND == LOG) {
    return r2 > 0.0 ? 0.5 * log(r2) : 0.0;
  } else if constexpr (KIND == REG_INVERSE) {
    double r = sqrt(r2);
    return r < kp.a ? r / kp.a : kp.a / r;
  } else {  // REG_LOG
    double r = sqrt(r2);
    if (r >= kp.a) return log(r) * kp.inv_log_a;
    if (r == 0.0) return 0.0;
    return r * (log(r) - 1.0) * kp.c_near;
  }
}

template <int KIND>
__host__ __device__ constexpr double kscale() {
  return KIND == LAPLACE ? INV_FOUR_PI : 1.0;
}

__global__ void gather_rows(const double* __restrict__ w, const int64_t* __restrict__ perm, int64_t n, int64_t R,
                            double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * R) return;
  int64_t p = i / R, r = i - p * R;
  out[i] = w[perm[p] * R + r];
}

// upward: y_c[s] = sum_j A_c[s*nrow + j] x_c[j]   (P2M, M2M; A = column interpolator)
// one CTA per cell, one warp per output row s
__global__ void gemv_t(int64_t ncell, const int64_t* __restrict__ kout, const int64_t* __restrict__ nrow,
                       const double* __restrict__ A, const int64_t* __restrict__ a_off,
                       const double* __restrict__ x, const int64_t* __restrict__ x_ptr,
                       const int64_t* __restrict__ x_map, double* __restrict__ y, const int64_t* __restrict__ y_ptr,
                       int64_t R) {
  int64_t c = blockIdx.x;
  if (c >= ncell) return;
  const int64_t k = kout[c], nr = nrow[c];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t xo = x_map ? x_ptr[x_map[c]] : x_ptr[c];
  const double* Ac = A + a_off[c];
  const double* xc = x + xo * R;
  double* yc = y + y_ptr[c] * R;
  for (int64_t s = warp; s < k; s += nw) {
    const double* As = Ac + s * nr;
    for (int64_t r = 0; r < R; r++) {
      double acc = 0.0;
      for (int64_t j = lane; j < nr; j += 32) acc = fma(As[j], xc[j * R + r], acc);
      acc = warp_sum(acc);
      if (lane == 0) yc[s * R + r] = acc;
    }
  }
}

// downward: y_c[i] += sum_s A_c[s*nrow + i] x_c[s]   (L2L; A = row interpolator)
__global__ void gemv_n_add(int64_t ncell, const int64_t* __restrict__ kin, const int64_t* __restrict__ nrow,
                           const double* __restrict__ A, const int64_t* __restrict__ a_off,
                           const double* __restrict__ x, const int64_t* __restrict__ x_ptr, double* __restrict__ y,
                           const int64_t* __restrict__ y_ptr, const int64_t* __restrict__ y_map, int64_t R) {
  int64_t c = blockIdx.x;
  if (c >= ncell) return;
  const int64_t k = kin[c], nr = nrow[c];
  const double* Ac = A + a_off[c];
  const double* xc = x + x_ptr[c] * R;
  double* yc = y + y_ptr[y_map[c]] * R;
  for (int64_t i = threadIdx.x; i < nr; i += blockDim.x)
    for (int64_t r = 0; r < R; r++) {
      double acc = 0.0;
      for (int64_t s = 0; s < k; s++) acc = fma(Ac[s * nr + i], xc[s * R + r], acc);
      yc[i * R + r] += acc;
    }
}

constexpr int IT = 128;  // interaction kernel threads

struct Interact {
  // targets
  const double* tc;  // SoA, ld_t
  int64_t ld_t;
  const int64_t* t_ptr;  // target range per cell
  // sources
  const double* sc;  // SoA, ld_s
  int64_t ld_s;
  const int64_t* s_ptr;  // source range per source cell
  const double* q;       // charges (ld R)
  // list
  const int64_t* l_ptr;
  const int64_t* l_idx;
  // output
  double* out;              // indexed by (target position) * R + r
  const int64_t* out_perm;  // if set: out row = out_perm[target position]
  // optional fused L2P: out += P_c (m x k, col-major) * uin_c
  const double* pm;
  const int64_t* pm_off;
  const int64_t* kin;
  const int64_t* in_ptr;
  const double* uin;
  int64_t R, r0;
  KParams kp;
};

// Sum over the cell list of K(target, source) * charge, with NR right-hand
// sides at once.  Thread = (target slot, source group); groups stride the
// list members; sources are read straight from L1/L2 as warp broadcasts.
template <int D, int KIND, int NR>
__global__ void __launch_bounds__(IT) interact_kernel(Interact P) {
  __shared__ double part[IT * NR];
  const int64_t c = blockIdx.x;
  const int64_t tb = P.t_ptr[c], m = P.t_ptr[c + 1] - tb;
  if (m == 0) return;
  const int64_t lb = P.l_ptr[c], le = P.l_ptr[c + 1];
  int TS = 1;
  while (TS < m && TS < IT) TS <<= 1;
  const int G = IT / TS;
  const int slot = threadIdx.x % TS, grp = threadIdx.x / TS;
  for (int64_t a0 = 0; a0 < m; a0 += TS) {
    const int64_t a = a0 + slot;
    const bool active = a < m;
    double x[D];
#pragma unroll
    for (int k = 0; k < D; k++) x[k] = active ? P.tc[k * P.ld_t + tb + a] : 0.0;
    double acc[NR];
#pragma unroll
    for (int r = 0; r < NR; r++) acc[r] = 0.0;
    if (active) {
      for (int64_t q = lb + grp; q < le; q += G) {
        const int64_t sc = P.l_idx[q];
        const int64_t sb = P.s_ptr[sc], se = P.s_ptr[sc + 1];
        int64_t j = sb;
        for (; j + 1 < se; j += 2) {
          double r2a = 0.0, r2b = 0.0;
#pragma unroll
          for (int k = 0; k < D; k++) {
            double da = x[k] - __ldg(P.sc + k * P.ld_s + j);
            double db = x[k] - __ldg(P.sc + k * P.ld_s + j + 1);
            r2a = fma(da, da, r2a);
            r2b = fma(db, db, r2b);
          }
          double ka = kfast<KIND>(r2a, P.kp), kb = kfast<KIND>(r2b, P.kp);
#pragma unroll
          for (int r = 0; r < NR; r++) {
            acc[r] = fma(ka, __ldg(P.q + j * P.R + P.r0 + r), acc[r]);
            acc[r] = fma(kb, __ldg(P.q + (j + 1) * P.R + P.r0 + r), acc[r]);
          }
        }
        if (j < se) {
          double r2a = 0.0;
#pragma unroll
          for (int k = 0; k < D; k++) {
            double da = x[k] - __ldg(P.sc + k * P.ld_s + j);
            r2a = fma(da, da, r2a);
          }
          double ka = kfast<KIND>(r2a, P.kp);
#pragma unroll
          for (int r = 0; r < NR; r++) acc[r] = fma(ka, __ldg(P.q + j * P.R + P.r0 + r), acc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < NR; r++) part[threadIdx.x * NR + r] = acc[r];
    __syncthreads();
    if (grp == 0 && active) {
      double tot[NR];
#pragma unroll
      for (int r = 0; r < NR; r++) tot[r] = 0.0;
      for (int g = 0; g < G; g++)
#pragma unroll
        for (int r = 0; r < NR; r++) tot[r] += part[(g * TS + slot) * NR + r];
#pragma unroll
      for (int r = 0; r < NR; r++) tot[r] *= kscale<KIND>();
      if (P.pm) {  // fused L2P
        const int64_t k = P.kin[c];
        const double* Pc = P.pm + P.pm_off[c];
        const double* uc = P.uin + P.in_ptr[c] * P.R;
        for (int64_t s = 0; s < k; s++) {
          double pv = Pc[s * m + a];
#pragma unroll
          for (int r = 0; r < NR; r++) tot[r] = fma(pv, uc[s * P.R + P.r0 + r], tot[r]);
        }
      }
      const int64_t row = P.out_perm ? P.out_perm[tb + a] : tb + a;
#pragma unroll
      for (int r = 0; r < NR; r++) P.out[row * P.R + P.r0 + r] = tot[r];
    }
    __syncthreads();
  }
}

template <int D, int KIND>
void launch_interact_k(const Interact& P, int64_t ncell, int nr, cudaStream_t s) {
  switch (nr) {
    case 16: interact_kernel<D, KIND, 16><<<(unsigned)ncell, IT, 0, s>>>(P); break;
    case 8: interact_kernel<D, KIND, 8><<<(unsigned)ncell, IT, 0, s>>>(P); break;
    case 4: interact_kernel<D, KIND, 4><<<(unsigned)ncell, IT, 0, s>>>(P); break;
    case 2: interact_kernel<D, KIND, 2><<<(unsigned)ncell, IT, 0, s>>>(P); break;
    default: interact_kernel<D, KIND, 1><<<(unsigned)ncell, IT, 0, s>>>(P); break;
  }
  CKL();
}

template <int D>
void launch_interact(int kind, const Interact& P, int64_t ncell, int nr, cudaStream_t s) {
  if (ncell == 0) return;
  switch (kind) {
    case COULOMB: launch_interact_k<D, COULOMB>(P, ncell, nr, s); break;
    case LAPLACE: launch_interact_k<D, LAPLACE>(P, ncell, nr, s); break;
    case GAUSSIAN: launch_interact_k<D, GAUSSIAN>(P, ncell, nr, s); break;
    case GAUSSIAN_SCALED: launch_interact_k<D, GAUSSIAN_SCALED>(P, ncell, nr, s); break;
    case MATERN: launch_interact_k<D, MATERN>(P, ncell, nr, s); break;
    case LOG: launch_interact_k<D, LOG>(P, ncell, nr, s); break;
    case REG_INVERSE: launch_interact_k<D, REG_INVERSE>(P, ncell, nr, s); break;
    default: launch_interact_k<D, REG_LOG>(P, ncell, nr, s); break;
  }
}

void interact(int d, int kind, const Interact& P, int64_t ncell, int nr, cudaStream_t s) {
  switch (d) {
    case 1: launch_interact<1>(kind, P, ncell, nr, s); break;
    case 2: launch_interact<2>(kind, P, ncell, nr, s); break;
    case 3: launch_interact<3>(kind, P, ncell, nr, s); break;
    default: launch_interact<4>(kind, P, ncell, nr, s); break;
  }
}

KParams make_kp(int kind, double a) {
  KParams kp;
  kp.a = a;
  kp.inv_log_a = 0;
  kp.c_near = 0;
  if (kind == REG_LOG) {
    kp.inv_log_a = 1.0 / std::log(a);
    kp.c_near = 1.0 / (a * (std::log(a) - 1.0));
  }
  return kp;
}

void ensure_scratch(DevH2& h, int64_t R) {
  const DevTree& T = *h.t;
  if (h.scratch_nrhs == R) return;
  h.w_sorted.alloc(T.nq * R);
  h.wout.clear();
  h.uin.clear();
  h.wout.resize(T.depth + 1);
  h.uin.resize(T.depth + 1);
  for (int l = 2; l <= T.depth; l++) {
    h.wout[l].alloc(std::max<int64_t>(h.lv[l].out_total * R, 1));
    h.uin[l].alloc(std::max<int64_t>(h.lv[l].in_total * R, 1));
  }
  h.scratch_nrhs = R;
}

// 1D-chunked RHS widths supported by the interaction kernel
void rhs_chunks(int64_t R, std::vector<std::pair<int64_t, int>>& out) {
  out.clear();
  int64_t r0 = 0;
  while (r0 < R) {
    int64_t left = R - r0;
    int nr = left >= 16 ? 16 : left >= 8 ? 8 : left >= 4 ? 4 : left >= 2 ? 2 : 1;
    out.push_back({r0, nr});
    r0 += nr;
  }
}

}  // namespace

void set_profiling(bool on) { g_profile = on; }
void last_stage_ms(double* ms5) {
  for (int i = 0; i < 5; i++) ms5[i] = g_stage_ms[i];
}

int64_t matvec_launches(const DevH2& h, int64_t nrhs) {
  const int L = h.t->depth;
  std::vector<std::pair<int64_t, int>> ch;
  rhs_chunks(nrhs, ch);
  int64_t nchunk = (int64_t)ch.size();
  if (L < 2) return 1 + nchunk;
  return 1 + 1 + (L - 2) + (L - 1) * nchunk + (L - 2) + nchunk;
}

void matvec(DevH2& h, const double* w, double* u, int64_t R, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth, d = T.d;
  ensure_scratch(h, R);
  KParams kp = make_kp(h.kind, h.a);
  std::vector<std::pair<int64_t, int>> chunks;
  rhs_chunks(R, chunks);
  cudaEvent_t ev[5];
  if (g_profile) {
    for (auto& e : ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ev[0], s));
  }
  gather_rows<<<ceil_div(T.nq * R, 256), 256, 0, s>>>(w, T.sperm(), T.nq, R, h.w_sorted.get());
  CKL();
  if (L >= 2) {
    // ---- upward pass: P2M at the leaves, then M2M ----
    {
      const DevLevel& Lv = T.lv[L];
      const DevH2Level& HL = h.lv[L];
      gemv_t<<<(unsigned)Lv.n, 128, 0, s>>>(Lv.n, HL.koutd(), HL.n_outd(), HL.qmatd(), HL.qm_offd(),
                                            h.w_sorted.get(), T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get(), nullptr,
                                            h.wout[L].get(), HL.out_ptrd(), R);
      CKL();
    }
    for (int l = L - 1; l >= 2; l--) {
      const DevLevel& Lv = T.lv[l];
      const DevH2Level& HL = h.lv[l];
      const DevH2Level& HC = h.lv[l + 1];
      gemv_t<<<(unsigned)Lv.n, 128, 0, s>>>(Lv.n, HL.koutd(), HL.n_outd(), HL.qmatd(), HL.qm_offd(),
                                            h.wout[l + 1].get(), HC.out_ptrd(), Lv.ch_ptr.get(), h.wout[l].get(),
                                            HL.out_ptrd(), R);
      CKL();
    }
    if (g_profile) CK(cudaEventRecord(ev[1], s));
    // ---- transverse pass (M2L), every level ----
    for (int l = 2; l <= L; l++) {
      const DevLevel& Lv = T.lv[l];
      const DevH2Level& HL = h.lv[l];
      Interact P{};
      P.tc = HL.tin_c.get();
      P.ld_t = std::max<int64_t>(HL.in_total, 1);
      P.t_ptr = HL.in_ptr.get();
      P.sc = HL.sout_cd();
      P.ld_s = std::max<int64_t>(HL.out_total, 1);
      P.s_ptr = HL.out_ptrd();
      P.q = h.wout[l].get();
      P.l_ptr = Lv.il_ptr.get();
      P.l_idx = Lv.il_idx.get();
      P.out = h.uin[l].get();
      P.R = R;
      P.kp = kp;
      for (auto& ch : chunks) {
        P.r0 = ch.first;
        interact(d, h.kind, P, Lv.n, ch.second, s);
      }
    }
    if (g_profile) CK(cudaEventRecord(ev[2], s));
    // ---- downward pass (L2L) ----
    for (int l = 2; l < L; l++) {
      const DevLevel& Lv = T.lv[l];
      const DevH2Level& HL = h.lv[l];
      const DevH2Level& HC = h.lv[l + 1];
      gemv_n_add<<<(unsigned)Lv.n, 128, 0, s>>>(Lv.n, HL.kin.get(), HL.m_in.get(), HL.pmat.get(), HL.pm_off.get(),
                                                h.uin[l].get(), HL.in_ptr.get(), h.uin[l + 1].get(), HC.in_ptr.get(),
                                                Lv.ch_ptr.get(), R);
      CKL();
    }
  } else if (g_profile) {
    CK(cudaEventRecord(ev[1], s));
    CK(cudaEventRecord(ev[2], s));
  }
  if (g_profile) CK(cudaEventRecord(ev[3], s));
  // ---- near field (P2P) + L2P + scatter to the caller's order ----
  {
    const DevLevel& Lv = T.lv[L];
    Interact P{};
    P.tc = T.tsd();
    P.ld_t = T.np;
    P.t_ptr = Lv.t_ptr.get();
    P.sc = T.ssd();
    P.ld_s = T.nq;
    P.s_ptr = T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get();
    P.q = h.w_sorted.get();
    P.l_ptr = Lv.nb_ptr.get();
    P.l_idx = Lv.nb_idx.get();
    P.out = u;
    P.out_perm = T.t_perm.get();
    if (L >= 2) {
      const DevH2Level& HL = h.lv[L];
      P.pm = HL.pmat.get();
      P.pm_off = HL.pm_off.get();
      P.kin = HL.kin.get();
      P.in_ptr = HL.in_ptr.get();
      P.uin = h.uin[L].get();
    }
    P.R = R;
    P.kp = kp;
    for (auto& ch : chunks) {
      P.r0 = ch.first;
      interact(d, h.kind, P, Lv.n, ch.second, s);
    }
  }
  if (g_profile) {
    CK(cudaEventRecord(ev[4], s));
    CK(cudaEventSynchronize(ev[4]));
    float t;
    CK(cudaEventElapsedTime(&t, ev[0], ev[1]));
    g_stage_ms[0] = t;
    CK(cudaEventElapsedTime(&t, ev[1], ev[2]));
    g_stage_ms[1] = t;
    CK(cudaEventElapsedTime(&t, ev[2], ev[3]));
    g_stage_ms[2] = t;
    CK(cudaEventElapsedTime(&t, ev[3], ev[4]));
    g_stage_ms[3] = t;
    CK(cudaEventElapsedTime(&t, ev[0], ev[4]));
    g_stage_ms[4] = t;
    for (auto& e : ev) cudaEventDestroy(e);
  }
}

// ---------------------------------------------------------------------
// dense oracles (matvec.py:574 dense_matvec) and kernel blocks
// ---------------------------------------------------------------------
namespace {

template <int D>
__global__ void dense_kernel(int kind, double a, const double* __restrict__ P, int64_t np,
                             const int64_t* __restrict__ rows, const double* __restrict__ Q, int64_t nq,
                             const double* __restrict__ w, double* __restrict__ u, int64_t R) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= np) return;
  const int64_t pi = rows ? rows[i] : i;
  double x[D];
#pragma unroll
  for (int k = 0; k < D; k++) x[k] = P[pi * D + k];
  for (int64_t r = 0; r < R; r++) {
    double acc = 0.0;
    for (int64_t j = 0; j < nq; j++) {
      double y[D];
#pragma unroll
      for (int k = 0; k < D; k++) y[k] = __ldg(Q + j * D + k);
      acc = fma(kval_exact(kind, a, r2_exact<D>(x, y)), __ldg(w + j * R + r), acc);
    }
    u[i * R + r] = acc;
  }
}

template <int D>
__global__ void block_kernel(int kind, double a, const double* __restrict__ X, int64_t m,
                             const double* __restrict__ Y, int64_t n, double* __restrict__ out) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= m * n) return;
  int64_t i = q / n, j = q - i * n;
  double x[D], y[D];
#pragma unroll
  for (int k = 0; k < D; k++) {
    x[k] = X[i * D + k];
    y[k] = Y[j * D + k];
  }
  out[q] = kval_exact(kind, a, r2_exact<D>(x, y));
}

}  // namespace

void dense_matvec(int kind, double a, const double* P, int64_t np, const double* Q, int64_t nq, int d,
                  const double* w, double* u, int64_t R, cudaStream_t s) {
  unsigned g = ceil_div(np, 128);
  switch (d) {
    case 1: dense_kernel<1><<<g, 128, 0, s>>>(kind, a, P, np, nullptr, Q, nq, w, u, R); break;
    case 2: dense_kernel<2><<<g, 128, 0, s>>>(kind, a, P, np, nullptr, Q, nq, w, u, R); break;
    case 3: dense_kernel<3><<<g, 128, 0, s>>>(kind, a, P, np, nullptr, Q, nq, w, u, R); break;
    default: dense_kernel<4><<<g, 128, 0, s>>>(kind, a, P, np, nullptr, Q, nq, w, u, R); break;
  }
  CKL();
}

void dense_rows_dev(int kind, double a, const double* P, const int64_t* rows, int64_t nrows, const double* Q,
                    int64_t nq, int d, const double* w, double* u, cudaStream_t s) {
  unsigned g = ceil_div(nrows, 128);
  switch (d) {
    case 1: dense_kernel<1><<<g, 128, 0, s>>>(kind, a, P, nrows, rows, Q, nq, w, u, 1); break;
    case 2: dense_kernel<2><<<g, 128, 0, s>>>(kind, a, P, nrows, rows, Q, nq, w, u, 1); break;
    case 3: dense_kernel<3><<<g, 128, 0, s>>>(kind, a, P, nrows, rows, Q, nq, w, u, 1); break;
    default: dense_kernel<4><<<g, 128, 0, s>>>(kind, a, P, nrows, rows, Q, nq, w, u, 1); break;
  }
  CKL();
}

void kernel_block(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d, double* out,
                  cudaStream_t s) {
  if (m * n == 0) return;
  unsigned g = ceil_div(m * n, 256);
  switch (d) {
    case 1: block_kernel<1><<<g, 256, 0, s>>>(kind, a, X, m, Y, n, out); break;
    case 2: block_kernel<2><<<g, 256, 0, s>>>(kind, a, X, m, Y, n, out); break;
    case 3: block_kernel<3><<<g, 256, 0, s>>>(kind, a, X, m, Y, n, out); break;
    default: block_kernel<4><<<g, 256, 0, s>>>(kind, a, X, m, Y, n, out); break;
  }
  CKL();
}

// FP64 FMA throughput probe: 8 independent DFMA chains per thread, full chip.
namespace {
__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1234.5) out[0] = s;
}
}  // namespace

double fp64_peak_tflops(cudaStream_t s) {
  int dev = 0, nsm = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  DBuf<double> out;
  out.alloc(1);
  const int threads = 512, blocks = nsm * 4, iters = 4096;
  dfma_peak_kernel<<<blocks, threads, 0, s>>>(out.get(), 64, 0.999999, 1e-7);  // warm-up
  CKL();
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  dfma_peak_kernel<<<blocks, threads, 0, s>>>(out.get(), iters, 0.999999, 1e-7);
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  return flops / (ms * 1e-3) / 1e12;
}

}  // namespace h2b
