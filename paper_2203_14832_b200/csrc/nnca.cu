// nnca.cu — NNCA construction on the GPU (compress.py:216 select_pivots,
// compress.py:285 assemble) with the partially pivoted ACA of
// _accel/_core.pyx:70 run by persistent CTAs (one cell at a time each, cells
// pulled from a work queue), level-batched bottom-up.
//
// Pivot parity: every residual entry is formed with the reference's exact
// operation order (kernel value, then `acc -= U[i,t] * V[j,t]` for t =
// 0..k-1, no FMA), so residual rows/columns are bitwise identical to the
// reference's and the argmax pivot choices (ties -> lowest index) agree.
// Only the Frobenius-norm bookkeeping for the stopping test is a parallel
// reduction (different summation order), which can flip the stop decision
// only when ||u_k|| ||v_k|| lands within roundoff of eps ||A_k||_F.
//
// Interpolation operators (aca.py:297 row_interpolator, :311
// col_interpolator) are back-substitutions against the pivot rows of U / V
// — the ACA byproduct, no further kernel evaluations (paper Remark 2).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"

namespace h2b {

namespace {

// ring configurations of the persistent ACA kernel (threads per CTA, columns per thread, rows per batch, CTAs
// per SM): the wide one (levels with few cells) and the small one (levels with >= H2B_ACA_CELLS_S cells); a
// 256-thread configuration sits between them (run_side)
#ifndef H2B_ACA_NT
#define H2B_ACA_NT 512
#endif
#ifndef H2B_ACA_NC
#define H2B_ACA_NC 4
#endif
#ifndef H2B_ACA_TB
#define H2B_ACA_TB 4
#endif
#ifndef H2B_ACA_MINB
#define H2B_ACA_MINB 1
#endif
#ifndef H2B_ACA_NT_S
#define H2B_ACA_NT_S 128
#endif
#ifndef H2B_ACA_NC_S
#define H2B_ACA_NC_S 4
#endif
#ifndef H2B_ACA_TB_S
#define H2B_ACA_TB_S 4
#endif
#ifndef H2B_ACA_MB_S
#define H2B_ACA_MB_S 4
#endif
#ifndef H2B_ACA_CELLS_S
#define H2B_ACA_CELLS_S 2400  // levels with at least this many cells use the small-CTA configuration
#endif
#ifndef H2B_ACA_CELLS_M
#define H2B_ACA_CELLS_M 600   // ... this many: 256-thread CTAs, two per SM; fewer: one 512-thread CTA per SM
#endif
#ifndef H2B_ACA_SLOTS
#define H2B_ACA_SLOTS 4  // ring depth wanted (bounded by shared memory and ACA_MAX_SLOTS)
#endif
#ifndef H2B_ACA_UPREF
#define H2B_ACA_UPREF 512  // doubles of shared memory kept for U before the ring takes the rest
#endif
#ifndef H2B_ACA_SLAB_PAD
#define H2B_ACA_SLAB_PAD 544
#endif

constexpr int ACA_MAX_THREADS = 1024;
constexpr int ACA_MAX_WARPS = ACA_MAX_THREADS / 32;
constexpr int XCH = 8;  // cross-product partial sums per pass
constexpr int ACA_MAX_SLOTS = 6;
// used-row / used-column bit masks in static shared memory: rows + columns up to ~65K per cell; the wide
// configuration (upper levels, rank caps in the hundreds) keeps its shared memory for the per-warp vectors
constexpr int aca_bit_words(int nt) { return nt >= 512 ? 512 : 2048; }

struct AcaArgs {
  int kind;
  double a, eps2;
  int64_t cell0;
  const int64_t *m, *n, *cap;
  const double* row_base;
  int64_t ld_row;
  const int64_t* row_off;
  const int64_t* row_gidx;
  const double* col_base;
  int64_t ld_col;
  const int64_t* col_off;
  const int64_t* col_gidx;
  double* U;
  const int64_t* u_off;
  double* V;
  const int64_t* v_off;
  unsigned char* flags;
  const int64_t* f_off;
  const int64_t* piv_off;
  int64_t *rp, *cp;        // local pivots (staging, at piv_off)
  int64_t *tpiv, *spiv;    // global pivot indices (staging, at piv_off)
  int64_t *rank, *conv, *nevals;
};

struct RedScratch {
  double v[ACA_MAX_WARPS];
  long long i[ACA_MAX_WARPS];
  double x[ACA_MAX_WARPS][XCH];
  double bv;     // block result (value)
  long long bi;  // block result (index)
};

// Block reductions: warp shuffles, then warp 0 reduces the per-warp results
// and broadcasts through shared memory (two barriers).
template <int NT>
__device__ void block_argmax(double& v, int64_t& i, RedScratch& rs) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  warp_argmax_nn(v, i);  // candidates are |residual| >= 0, indices < 2^31 (checked on the host)
  if (lane == 0) {
    rs.v[w] = v;
    rs.i[w] = i;
  }
  __syncthreads();
  if (w == 0) {
    double v2 = lane < NW ? rs.v[lane] : -1.0;
    int64_t i2 = lane < NW ? (int64_t)rs.i[lane] : -1;
    warp_argmax_nn(v2, i2);
    if (lane == 0) {
      rs.bv = v2;
      rs.bi = i2;
    }
  }
  __syncthreads();
  v = rs.bv;
  i = rs.bi;
}

// argmax (non-negative candidates, ties to the lowest index) and a sum in one pass: two barriers instead of four
template <int NT>
__device__ double block_argmax_sum(double& v, int64_t& i, double x, RedScratch& rs) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  warp_argmax_nn(v, i);
  x = warp_sum(x);
  if (lane == 0) {
    rs.v[w] = v;
    rs.i[w] = i;
    rs.x[w][0] = x;
  }
  __syncthreads();
  if (w == 0) {
    double v2 = lane < NW ? rs.v[lane] : -1.0;
    int64_t i2 = lane < NW ? (int64_t)rs.i[lane] : -1;
    warp_argmax_nn(v2, i2);
    if (lane == 0) {
      rs.bv = v2;
      rs.bi = i2;
      double s2 = 0.0;  // fixed left-to-right order over warps, as block_sum
      for (int q = 0; q < NW; q++) s2 += rs.x[q][0];
      rs.x[0][1] = s2;
    }
  }
  __syncthreads();
  v = rs.bv;
  i = rs.bi;
  return rs.x[0][1];
}

template <int NT>
__device__ double block_sum(double x, RedScratch& rs) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  x = warp_sum(x);
  if (lane == 0) rs.v[w] = x;
  __syncthreads();
  if (w == 0) {
    // fixed left-to-right order over warps (deterministic)
    double s2 = 0.0;
    if (lane == 0)
      for (int q = 0; q < NW; q++) s2 += rs.v[q];
    if (lane == 0) rs.bv = s2;
  }
  __syncthreads();
  return rs.bv;
}

template <int NT>
__device__ int64_t block_min(int64_t x, RedScratch& rs) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  x = warp_min_i64(x);
  if (lane == 0) rs.i[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t y = lane < NW ? (int64_t)rs.i[lane] : INT64_MAX;
    y = warp_min_i64(y);
    if (lane == 0) rs.bi = y;
  }
  __syncthreads();
  return rs.bi;
}

// _core.pyx:70-191, one CTA per cell
template <int D, int NT>
__global__ void __launch_bounds__(NT, (2048 / NT / 2) > 0 ? (2048 / NT / 2) : 1) aca_kernel(AcaArgs A) {
  constexpr int ACA_THREADS = NT;
  constexpr int ACA_WARPS = NT / 32;
  extern __shared__ double sm[];
  __shared__ RedScratch rs;
  __shared__ double xt[D], yb[D];
  const int64_t cell = A.cell0 + blockIdx.x;
  const int64_t m = A.m[cell], n = A.n[cell], cap = A.cap[cell];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (m == 0 || n == 0 || cap == 0) {
    if (tid == 0) {
      A.rank[cell] = 0;
      A.conv[cell] = (m == 0 || n == 0) ? 1 : 0;
      A.nevals[cell] = 0;
    }
    return;
  }
  double* urow = sm;
  double* vcol = sm + cap;
  double* crossv = sm + 2 * cap;
  double* crossu = sm + 3 * cap;
  const double* Xb = A.row_base + A.row_off[cell];
  const double* Yb = A.col_base + A.col_off[cell];
  const int64_t ldr = A.ld_row, ldc = A.ld_col;
  double* U = A.U + A.u_off[cell];
  double* V = A.V + A.v_off[cell];
  unsigned char* ru = A.flags + A.f_off[cell];
  unsigned char* cu = ru + m;
  int64_t* rp = A.rp + A.piv_off[cell];
  int64_t* cp = A.cp + A.piv_off[cell];
  for (int64_t q = tid; q < m + n; q += ACA_THREADS) ru[q] = 0;
  const int64_t full = m < n ? m : n;
  int64_t k = 0, trial = 0, nev = 0;
  double norm2 = 0.0;
  int64_t converged = 1;
  __syncthreads();
  for (;;) {
    bool exhausted = false;
    double best;
    int64_t bj;
    for (;;) {
      if (tid == 0) ru[trial] = 1;
      for (int64_t t = tid; t < k; t += ACA_THREADS) urow[t] = U[t * m + trial];
      if (tid < D) xt[tid] = Xb[tid * ldr + trial];
      __syncthreads();
      double xl[D];
#pragma unroll
      for (int q = 0; q < D; q++) xl[q] = xt[q];
      best = -1.0;
      bj = -1;
      // two columns per thread per pass: two independent exact-order chains
      // keep twice the V loads in flight (the pass is DRAM-latency bound)
      for (int64_t j0 = tid; j0 < n; j0 += 2 * ACA_THREADS) {
        const int64_t j1 = j0 + ACA_THREADS;
        const bool has1 = j1 < n;
        double y0[D], y1[D];
#pragma unroll
        for (int q = 0; q < D; q++) {
          y0[q] = Yb[q * ldc + j0];
          y1[q] = has1 ? Yb[q * ldc + j1] : y0[q];
        }
        double acc0 = kval_exact(A.kind, A.a, r2_exact<D>(xl, y0));
        double acc1 = kval_exact(A.kind, A.a, r2_exact<D>(xl, y1));
        const double* V0 = V + j0;
        const double* V1 = V + (has1 ? j1 : j0);
#pragma unroll 8
        for (int64_t t = 0; t < k; t++) {
          const double ut = urow[t];
          acc0 = __dsub_rn(acc0, __dmul_rn(ut, V0[t * n]));
          acc1 = __dsub_rn(acc1, __dmul_rn(ut, V1[t * n]));
        }
        V[k * n + j0] = acc0;
        if (!cu[j0]) {
          const double val = fabs(acc0);
          if (val > best) {
            best = val;
            bj = j0;
          }
        }
        if (has1) {
          V[k * n + j1] = acc1;
          if (!cu[j1]) {
            const double val = fabs(acc1);
            if (val > best) {
              best = val;
              bj = j1;
            }
          }
        }
      }
      if (bj < 0) best = -1.0;
      block_argmax<NT>(best, bj, rs);
      nev += n;
      if (best > 0.0) break;
      int64_t first = INT64_MAX;
      for (int64_t i = tid; i < m; i += ACA_THREADS)
        if (!ru[i] && i < first) first = i;
      first = block_min<NT>(first, rs);
      if (first == INT64_MAX) {
        exhausted = true;
        break;
      }
      trial = first;
      __syncthreads();
    }
    if (exhausted) break;
    const double piv = V[k * n + bj];
    __syncthreads();  // every thread holds piv before the owner of bj rescales it to 1
    double v2p = 0.0;
    for (int64_t j = tid; j < n; j += ACA_THREADS) {
      double v = __ddiv_rn(V[k * n + j], piv);
      V[k * n + j] = v;
      v2p += v * v;
    }
    if (tid < D) yb[tid] = Yb[tid * ldc + bj];
    __syncthreads();
    if (tid == 0) cu[bj] = 1;
    for (int64_t t = tid; t < k; t += ACA_THREADS) vcol[t] = V[t * n + bj];
    // crossv[t] = sum_j V[t][j] V[k][j]: threads keep their residual-row columns
    // j and XCH partial sums, so V is streamed once and V[k] only k/XCH times
    for (int64_t t0 = 0; t0 < k; t0 += XCH) {
      double ps[XCH];
#pragma unroll
      for (int c = 0; c < XCH; c++) ps[c] = 0.0;
      for (int64_t j = tid; j < n; j += ACA_THREADS) {
        const double vk = V[k * n + j];
#pragma unroll
        for (int c = 0; c < XCH; c++)
          if (t0 + c < k) ps[c] += V[(t0 + c) * n + j] * vk;
      }
#pragma unroll
      for (int c = 0; c < XCH; c++) {
        const double w = warp_sum(ps[c]);
        if (lane == 0) rs.x[warp][c] = w;
      }
      __syncthreads();
      if (tid < XCH && t0 + tid < k) {
        double w = 0.0;
        for (int q = 0; q < ACA_WARPS; q++) w += rs.x[q][tid];
        crossv[t0 + tid] = w;
      }
      __syncthreads();
    }
    double yl[D];
#pragma unroll
    for (int q = 0; q < D; q++) yl[q] = yb[q];
    double u2p = 0.0;
    for (int64_t i = tid; i < m; i += ACA_THREADS) {
      double xl[D];
#pragma unroll
      for (int q = 0; q < D; q++) xl[q] = Xb[q * ldr + i];
      double acc = kval_exact(A.kind, A.a, r2_exact<D>(xl, yl));
      for (int64_t t = 0; t < k; t++) acc = __dsub_rn(acc, __dmul_rn(U[t * m + i], vcol[t]));
      U[k * m + i] = acc;
      u2p += acc * acc;
    }
    nev += m;
    __syncthreads();
    for (int64_t t = warp; t < k; t += ACA_WARPS) {
      double s = 0.0;
      const double* Ut = U + t * m;
      const double* Uk = U + k * m;
      for (int64_t i = lane; i < m; i += 32) s += Ut[i] * Uk[i];
      s = warp_sum(s);
      if (lane == 0) crossu[t] = s;
    }
    double u2 = block_sum<NT>(u2p, rs);
    double v2 = block_sum<NT>(v2p, rs);  // block_sum syncs: crossu/crossv visible
    for (int64_t t = 0; t < k; t++) norm2 += 2.0 * crossu[t] * crossv[t];
    norm2 += u2 * v2;
    if (tid == 0) {
      rp[k] = trial;
      cp[k] = bj;
    }
    k += 1;
    int stop = 0;
    if (u2 * v2 <= A.eps2 * (norm2 > 0.0 ? norm2 : 0.0)) stop = 1;
    else if (k == full) stop = 1;
    else if (k == cap) stop = 2;
    if (stop) {
      if (stop == 2) converged = 0;
      break;
    }
    best = -1.0;
    int64_t bi = -1;
    const double* Uk = U + (k - 1) * m;
    for (int64_t i = tid; i < m; i += ACA_THREADS)
      if (!ru[i]) {
        double val = fabs(Uk[i]);
        if (val > best) {
          best = val;
          bi = i;
        }
      }
    block_argmax<NT>(best, bi, rs);
    if (bi < 0) break;
    trial = bi;
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    A.rank[cell] = k;
    A.conv[cell] = converged;
    A.nevals[cell] = nev;
  }
  for (int64_t t = tid; t < k; t += ACA_THREADS) {
    A.tpiv[A.piv_off[cell] + t] = A.row_gidx ? A.row_gidx[A.row_off[cell] + rp[t]] : rp[t];
    A.spiv[A.piv_off[cell] + t] = A.col_gidx ? A.col_gidx[A.col_off[cell] + cp[t]] : cp[t];
  }
}


// ---------------------------------------------------------------------
// candidate set sizing / gathering (compress.py:159 candidate_sets)
// ---------------------------------------------------------------------
struct Src {
  const double* coords;  // SoA, ld
  int64_t ld;
  const int64_t* gidx;   // global index per position
  const int64_t* ptr;    // per cell of the "owner" level: range via ptr[range_lo[c]] .. ptr[range_hi[c]]
  const int64_t* lo_map; // maps cell c -> index into ptr for begin (identity at leaf; ch_ptr otherwise)
};

// range of positions of cell c in the source: [ptr[map(c)], ptr[map(c+1)])
__device__ __forceinline__ void src_range(const Src& S, int64_t c, int64_t& b, int64_t& e) {
  if (S.lo_map) {
    b = S.ptr[S.lo_map[c]];
    e = S.ptr[S.lo_map[c + 1]];
  } else {
    b = S.ptr[c];
    e = S.ptr[c + 1];
  }
}

__global__ void cand_sizes(int64_t n, Src own, Src far, const int64_t* __restrict__ il_ptr,
                           const int64_t* __restrict__ il_idx, int64_t* own_b, int64_t* own_len,
                           int64_t* far_len) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  int64_t b, e;
  src_range(own, c, b, e);
  own_b[c] = b;
  own_len[c] = e - b;
  int64_t tot = 0;
  for (int64_t q = il_ptr[c]; q < il_ptr[c + 1]; q++) {
    src_range(far, il_idx[q], b, e);
    tot += e - b;
  }
  far_len[c] = tot;
}

// concatenate the far-field source ranges of each cell (IL order) into a
// contiguous SoA buffer (ld = total) with their global indices
template <int D>
__global__ void gather_far(int64_t cell0, Src far, const int64_t* __restrict__ il_ptr,
                           const int64_t* __restrict__ il_idx, const int64_t* __restrict__ dst_off,
                           double* __restrict__ dst, int64_t ld_dst, int64_t* __restrict__ dst_gidx) {
  const int64_t cell = cell0 + blockIdx.x;
  int64_t w = dst_off[cell];
  for (int64_t q = il_ptr[cell]; q < il_ptr[cell + 1]; q++) {
    int64_t b, e;
    src_range(far, il_idx[q], b, e);
    for (int64_t p = b + threadIdx.x; p < e; p += blockDim.x) {
      int64_t o = w + (p - b);
#pragma unroll
      for (int k = 0; k < D; k++) dst[k * ld_dst + o] = far.coords[k * far.ld + p];
      dst_gidx[o] = far.gidx[p];
    }
    w += e - b;
  }
}

template <int D>
__global__ void gather_coords(const double* __restrict__ aos, const int64_t* __restrict__ gidx, int64_t n,
                              double* __restrict__ soa) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t g = gidx[i];
#pragma unroll
  for (int k = 0; k < D; k++) soa[k * n + i] = aos[g * D + k];
}

__global__ void compact_pivots(int64_t n, const int64_t* __restrict__ rank, const int64_t* __restrict__ piv_off,
                               const int64_t* __restrict__ ptr, const int64_t* __restrict__ tp,
                               const int64_t* __restrict__ sp, int64_t* __restrict__ t_out,
                               int64_t* __restrict__ s_out) {
  int64_t c = blockIdx.x;
  if (c >= n) return;
  for (int64_t t = threadIdx.x; t < rank[c]; t += blockDim.x) {
    t_out[ptr[c] + t] = tp[piv_off[c] + t];
    s_out[ptr[c] + t] = sp[piv_off[c] + t];
  }
}

// compress.py:307-328 entry counts: sum_B kin(B) * sum_{C in IL(B)} kout(C)
__global__ void coupling_counts(int64_t n, const int64_t* __restrict__ kin, const int64_t* __restrict__ kout,
                                const int64_t* __restrict__ il_ptr, const int64_t* __restrict__ il_idx,
                                unsigned long long* out) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n || kin[c] == 0) return;
  int64_t s = 0;
  for (int64_t q = il_ptr[c]; q < il_ptr[c + 1]; q++) s += kout[il_idx[q]];
  atomicAdd(out, (unsigned long long)(s * kin[c]));
}

__global__ void near_counts(int64_t n, const int64_t* __restrict__ t_ptr, const int64_t* __restrict__ s_ptr,
                            const int64_t* __restrict__ nb_ptr, const int64_t* __restrict__ nb_idx,
                            unsigned long long* out) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  int64_t s = 0;
  for (int64_t q = nb_ptr[c]; q < nb_ptr[c + 1]; q++) {
    int64_t y = nb_idx[q];
    s += s_ptr[y + 1] - s_ptr[y];
  }
  atomicAdd(out, (unsigned long long)(s * (t_ptr[c + 1] - t_ptr[c])));
}

void excl_scan(const int64_t* in, int64_t n, int64_t* out_n1, cudaStream_t s) {
  DBuf<int64_t> tmpin;
  tmpin.alloc(n + 1);
  if (n) CK(cudaMemcpyAsync(tmpin.get(), in, n * 8, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemsetAsync(tmpin.get() + n, 0, 8, s));
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, tmpin.get(), out_n1, n + 1, s));
  DBuf<unsigned char> tmp;
  tmp.alloc(bytes);
  CK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, tmpin.get(), out_n1, n + 1, s));
  CK(cudaStreamSynchronize(s));
}

template <class T>
DBuf<T> upload(const std::vector<T>& h, cudaStream_t s, MemStats* ms = nullptr) {
  DBuf<T> d;
  d.alloc(std::max<size_t>(h.size(), 1), ms);
  if (!h.empty()) CK(cudaMemcpyAsync(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return d;
}

// ---------------------------------------------------------------------
// Persistent level-batched ACA (the setup hot path).
//
// CTAs pull cells from a work queue (largest first).  A CTA's workspace (the
// residual factors U, V, the positions of the far candidates in the level's
// source arrays) is a fixed per-CTA slab reused cell after cell.  Pivot arithmetic is the
// reference's (see aca_kernel): every residual entry is
//     K(x_i, y_j) - U[i,0] V[j,0] - ... - U[i,k-1] V[j,k-1]
// rounded after every multiply and every subtract, left to right.
//
// Row pass (the hot loop: step k re-reads all k previous residual rows):
// one thread owns NC columns of a column segment and keeps their running
// entries in registers, while the previous rows V[t][segment] stream through
// an S-slot shared-memory ring of TB rows each, filled by TMA bulk copies
// (cp.async.bulk, mbarrier completion; one copy per row, issued by thread 0
// S - 1 batches ahead, across segment and pass boundaries).  The copies keep
// TB rows x segment bytes in flight per slot with no registers held, which is
// what the latency-bound register version lacked (ncu: 16 warps,
// long-scoreboard stalls, 1.2 TB/s).  The
// pass also finishes step k - 1 (normalises its raw row, forms the cross
// products <V[t], V[k-1]> for the stopping test) so V is swept once per step.
// Kernel families (1/r-like, exp, log) are separate instantiations: the
// unused libm paths stay out of the loop (instruction-cache misses were 20%
// of the issue stalls with the runtime switch).
// ---------------------------------------------------------------------
enum KClass { KC_INV = 0, KC_EXP = 1, KC_LOG = 2 };
inline int kind_class(int kind) {
  switch (kind) {
    case COULOMB:
    case LAPLACE:
    case REG_INVERSE: return KC_INV;
    case GAUSSIAN:
    case GAUSSIAN_SCALED:
    case MATERN: return KC_EXP;
    default: return KC_LOG;
  }
}

// kval_exact restricted to one family (same operations, same roundings)
template <int KC>
__device__ __forceinline__ double kval_class(int kind, double a, double num, double r2) {
  if constexpr (KC == KC_INV) {  // num: numerator of the 1/r kernels (1 or 1/(4 pi)), hoisted by the caller
    const double r = __dsqrt_rn(r2);
    if (kind == REG_INVERSE) return r < a ? __ddiv_rn(r, a) : __ddiv_rn(a, r);
    return r == 0.0 ? 0.0 : __ddiv_rn(num, r);
  } else if constexpr (KC == KC_EXP) {
    if (kind == GAUSSIAN) return exp(-r2);
    if (kind == GAUSSIAN_SCALED) return exp(-__dmul_rn(a, r2));
    return exp(-__dsqrt_rn(r2));
  } else {
    if (kind == LOG) return kval_exact(LOG, a, r2);
    return kval_exact(REG_LOG, a, r2);
  }
}

#ifdef H2B_ACA_PROF
__device__ unsigned long long g_aca_prof[8];
#define APROF(i)                                                    \
  do {                                                              \
    __syncthreads();                                                \
    if (tid == 0) {                                                 \
      const long long now_ = clock64();                             \
      atomicAdd(&g_aca_prof[i], (unsigned long long)(now_ - last_)); \
      last_ = now_;                                                 \
    }                                                               \
  } while (0)
#else
#define APROF(i) \
  do {           \
  } while (0)
#endif

struct CellJob {
  int kind;
  double a, eps2;
  int64_t ncell;
  const int64_t* order;  // cells, largest first
  int rows_far;          // rows = far candidates (outgoing side) instead of own points
  Src own, far;
  const int64_t* il_ptr;
  const int64_t* il_idx;
  const int64_t* caps;
  const int64_t* piv_off;
  int64_t *tpiv, *spiv, *rank, *conv, *nevals;
  double* mat;
  const int64_t* mat_off;
  int which;  // 0: row interpolator from U (rows m); 1: column interpolator from V (rows n)
  double* ws;
  int64_t ws_doubles;  // per CTA
  int64_t f_max, cap_max;
  int64_t u_slab, v_slab;  // doubles reserved per CTA for U (cells whose U does not fit in shared memory) / V
  int64_t u_smem;          // doubles of shared memory for U: cells with cap x m <= u_smem keep U there
  int slots;               // ring depth (row batches of TB rows x one segment)
  int bit_words;           // > 0: used-row / used-column flags are bit masks in shared memory (else bytes in the slab)
  unsigned long long* counter;
};

// OUT: the outgoing side (rows = gathered far candidates, column interpolator from V) instead of the incoming
// one (rows = own points / children's pivots, row interpolator from U); a template parameter because the two
// sides' branches would otherwise sit in every loop of an instruction-cache-bound kernel.
template <int D, int KC, int NT, int NC, int TB, int MB, bool OUT>
__global__ void __launch_bounds__(NT, MB) aca_ring(CellJob J) {
  constexpr bool ROWS_FAR = OUT;
  constexpr int WHICH = OUT ? 1 : 0;
  static_assert(TB % 4 == 0, "row batches are reduced four rows at a time");
  constexpr int NW = NT / 32;
  constexpr int SEG = NT * NC;  // columns per segment (ring row length)
  extern __shared__ __align__(16) double sm[];
  __shared__ RedScratch rs;
  __shared__ double xt[D], yb[D];
  __shared__ long long s_cell;
  __shared__ int s_mp[NT + 1];   // member prefix (far gather; positions and counts are < 2^31, checked on the host)
  __shared__ int s_mb[NT];       // member range begin
  __shared__ __align__(8) uint64_t s_full[ACA_MAX_SLOTS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* ring = sm;  // [slots][TB][SEG]
  double* urow = ring + J.slots * (TB * SEG);
  double* vcol = urow + J.cap_max;
  double* crossv = vcol + J.cap_max;
  double* crossu = crossv + J.cap_max;
  double* crosspart = crossu + J.cap_max;  // [NW][cap]
  // used-row / used-column flags: bit masks in (static) shared memory when they fit (J.bit_words > 0), else bytes
  // in the slab
  __shared__ uint32_t s_bits[aca_bit_words(NT)];
  uint32_t* bits = s_bits;
  double* usm = crosspart + NW * J.cap_max;
  double* base = J.ws + (int64_t)blockIdx.x * J.ws_doubles;
  double* Ub = base;
  double* Vb = Ub + J.u_slab;
  // far candidates: their positions in the level's source arrays.  The coordinates are read through these from
  // the shared per-level arrays (each far point sits in the lists of ~80 cells, so those arrays stay L2-resident)
  // instead of from a private gathered copy per cell (24 bytes per candidate and pass of DRAM traffic)
  int* POS = reinterpret_cast<int*>(Vb + J.v_slab);
  int64_t* RP = reinterpret_cast<int64_t*>(POS + 2 * ((J.f_max + 1) / 2));
  int64_t* CP = RP + J.cap_max;
  unsigned char* flags = reinterpret_cast<unsigned char*>(CP + J.cap_max);
  const double knum = J.kind == LAPLACE ? INV_FOUR_PI : 1.0;
  const int S = J.slots;  // ring depth: S - 1 batches in flight while one is consumed
  if (tid == 0) {
    for (int q = 0; q < S; q++) mbar_init(&s_full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t bar0 = smem_u32(&s_full[0]), ring0 = smem_u32(ring);
  // stream state, uniform over the CTA: next slot to fill, slot to consume and its mbarrier parity, batches in
  // flight (issued, not yet consumed)
  int islot = 0, cslot = 0, inflight = 0;
  uint32_t cpar = 0;
  long long last_ = clock64();
  (void)last_;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      const unsigned long long q = atomicAdd(J.counter, 1ull);
      s_cell = q < (unsigned long long)J.ncell ? (long long)J.order[q] : -1ll;
    }
    __syncthreads();
    const int64_t cell = s_cell;
    if (cell < 0) break;
    // ---- own range and far candidates (gathered into the slab) ----
    int64_t ob, oe;
    src_range(J.own, cell, ob, oe);
    const int64_t own_n = oe - ob;
    const int64_t lb = J.il_ptr[cell], le = J.il_ptr[cell + 1];
    int64_t far_n = 0;
    for (int64_t q0 = lb; q0 < le; q0 += NT) {
      const int nm = (int)(le - q0 < NT ? le - q0 : NT);
      int64_t len = 0;
      if (tid < nm) {
        int64_t b, e;
        src_range(J.far, J.il_idx[q0 + tid], b, e);
        s_mb[tid] = (int)b;
        len = e - b;
      }
      int64_t v = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long n2 = __shfl_up_sync(0xffffffffu, (long long)v, o);
        if (lane >= o) v += n2;
      }
      if (lane == 31) rs.i[warp] = v;
      __syncthreads();
      int64_t off = far_n;
      for (int w = 0; w < warp; w++) off += rs.i[w];
      if (tid < nm) s_mp[tid + 1] = (int)(off + v);
      if (tid == 0) s_mp[0] = (int)far_n;
      int64_t tot = far_n;
      for (int w = 0; w < NW; w++) tot += rs.i[w];
      __syncthreads();
      for (int q = warp; q < nm; q += NW) {
        const int64_t b = s_mb[q], o0 = s_mp[q], len2 = s_mp[q + 1] - o0;
        for (int64_t e = lane; e < len2; e += 32) {
          POS[o0 + e] = (int)(b + e);
        }
      }
      far_n = tot;
      __syncthreads();
    }
    APROF(0);
    const int64_t m = ROWS_FAR ? far_n : own_n;
    const int64_t n = ROWS_FAR ? own_n : far_n;
    const int64_t cap = J.caps[cell];
    // row / column coordinate k of local index i
    auto rowc = [&](int k, int64_t i) -> double {
      return ROWS_FAR ? J.far.coords[k * J.far.ld + POS[i]] : J.own.coords[k * J.own.ld + ob + i];
    };
    auto colc = [&](int k, int64_t j) -> double {
      return ROWS_FAR ? J.own.coords[k * J.own.ld + ob + j] : J.far.coords[k * J.far.ld + POS[j]];
    };
    if (m == 0 || n == 0 || cap == 0) {
      if (tid == 0) {
        J.rank[cell] = 0;
        J.conv[cell] = (m == 0 || n == 0) ? 1 : 0;
        J.nevals[cell] = 0;
      }
      continue;
    }
    double* U = cap * m <= J.u_smem ? usm : Ub;  // U (cap x m) in shared memory when it fits
    double* V = Vb;                               // V (cap x ldv) in the slab, rows 16-byte aligned for the bulk copies
    const int ni = (int)n;
    const int64_t ldv = (n + 1) & ~(int64_t)1;
    const int nseg = (ni + SEG - 1) / SEG;
    const int seglen = (((ni + nseg - 1) / nseg) + 1) & ~1;
    unsigned char* ru = flags;
    unsigned char* cu = flags + m;
    const bool sbits = J.bit_words > 0;
    uint32_t* rbits = bits;
    uint32_t* cbits = bits + ((m + 31) >> 5);
    if (sbits) {
      for (int64_t q = tid; q < ((m + 31) >> 5) + ((n + 31) >> 5); q += NT) bits[q] = 0u;
    } else {
      for (int64_t q = tid; q < m + n; q += NT) ru[q] = 0;
    }
    auto row_used = [&](int i) -> bool { return sbits ? (rbits[i >> 5] >> (i & 31)) & 1u : ru[i] != 0; };
    auto col_used = [&](int j) -> bool { return sbits ? (cbits[j >> 5] >> (j & 31)) & 1u : cu[j] != 0; };
    const int64_t full = m < n ? m : n;
    int64_t k = 0, trial = 0, nev = 0;
    double norm2 = 0.0;
    int64_t converged = 1;
    __syncthreads();
    // Step k's row pass also finishes step k - 1 (fused, one sweep over V):
    // it normalises the raw residual row k - 1 (V[k-1] /= piv, written back),
    // forms crossv[t] = <V[t], V[k-1]> and |V[k-1]|^2, and only then is step
    // k - 1's stopping test evaluated -- the row pass of step k is
    // speculative and discarded (with its evaluation count) if step k - 1
    // stops.  Pivots, residual arithmetic and the test are unchanged; only the
    // summation order of the norm bookkeeping differs from the reference.
    bool pend = false;          // step k - 1 awaits normalisation + stopping test
    double piv_prev = 1.0, u2_prev = 0.0;
    // Batch q of a pass over kfq rows (nbq batches per segment): rows [b TB, b TB + TB) of segment q / nbq.
    // Thread 0 arms the slot's mbarrier and issues one bulk copy per row; every thread advances the stream state.
    int pre = 0;  // batches of the next pass already in flight
    int isg = 0, ib = 0;  // (segment, batch) of the next batch to issue: the stream is issued in order
    auto issue = [&](int q, int kfq, int nbq) {
      (void)q;
      if (tid == 0) {
        const int sg = isg, b = ib;
        const int c0 = sg * seglen;
        const int len = ni - c0 < seglen ? ni - c0 : seglen;
        const uint32_t bytes = (uint32_t)((len + 1) & ~1) * 8u;
        const int r0 = b * TB;
        const int rows = kfq - r0 < TB ? kfq - r0 : TB;
        const uint32_t bar = bar0 + 8u * (uint32_t)islot;
        mbar_expect_tx_u32(bar, (uint32_t)rows * bytes);
        const double* src = V + (int64_t)r0 * ldv + c0;
        const uint32_t dst = ring0 + (uint32_t)(islot * TB) * (uint32_t)(SEG * 8);
        for (int tt = 0; tt < rows; tt++) bulk_g2s_u32(dst + (uint32_t)tt * (uint32_t)(SEG * 8), src + (int64_t)tt * ldv, bytes, bar);
      }
      if (++ib == nbq) {  // the stream of a pass (and of the pass prefetched after it) runs segment by segment
        ib = 0;
        if (++isg == nseg) isg = 0;
      }
      if (++islot == S) islot = 0;
      inflight++;
    };
    // normalise row r = k - 1 on its own (and optionally its cross products): used when no fused pass follows
    auto finish_row = [&](int r, bool need_cross) -> double {
      double v2p = 0.0;
      double* Vr = V + (int64_t)r * ldv;
      for (int j = tid; j < ni; j += NT) {
        const double v = __ddiv_rn(Vr[j], piv_prev);
        Vr[j] = v;
        v2p += v * v;
      }
      __syncthreads();
      if (need_cross) {
        for (int t = warp; t < r; t += NW) {
          const double* Vt = V + (int64_t)t * ldv;
          double s0 = 0.0, s1 = 0.0;
          int j = lane;
          for (; j + 32 < ni; j += 64) {
            s0 = fma(Vt[j], Vr[j], s0);
            s1 = fma(Vt[j + 32], Vr[j + 32], s1);
          }
          for (; j < ni; j += 32) s0 = fma(Vt[j], Vr[j], s0);
          const double w = warp_sum(s0 + s1);
          if (lane == 0) crossv[t] = w;
        }
      }
      return block_sum<NT>(v2p, rs);  // syncs: crossv visible
    };
    for (;;) {
      bool exhausted = false, stop_prev = false, fuse = pend;
      double best;
      int64_t bj;
      for (;;) {
        if (tid == 0) {
          if (sbits) rbits[trial >> 5] |= 1u << (trial & 31);
          else ru[trial] = 1;
        }
        for (int64_t t = tid; t < k; t += NT) urow[t] = U[t * m + trial];
        if (tid < D) xt[tid] = rowc(tid, trial);
        if (fuse)
          for (int q = tid; q < NW * (int)cap; q += NT) crosspart[q] = 0.0;
        __syncthreads();
        double xl[D];
#pragma unroll
        for (int q = 0; q < D; q++) xl[q] = xt[q];
        best = -1.0;
        bj = -1;
        const int ki = (int)k;
        const int kf = fuse ? ki - 1 : ki;  // rows streamed (already normalised)
        const int nb = (kf + TB - 1) / TB;
        const int Q = nseg * nb;  // batches of this pass, streamed in (segment, batch) order
        int qi = pre;             // ... of which `pre` were issued at the end of the previous pass
        pre = 0;
        while (qi < Q && inflight < S) issue(qi++, kf, nb);
        double v2p = 0.0;
        double* Vlast = V + (int64_t)(ki - 1) * ldv;
        double* Vnew = V + (int64_t)ki * ldv;
        for (int sgi = 0; sgi < nseg; sgi++) {
          const int c0 = sgi * seglen;
          const int len = ni - c0 < seglen ? ni - c0 : seglen;
          double acc[NC], vl[NC];
          bool ok[NC];
          int off[NC];  // column offset inside a ring row; padding lanes read column 0 (finite, times vl = 0)
          {
            // all loads of the segment head first (coordinates, raw row k - 1), then the arithmetic
            double y[NC][D], raw[NC];
            int64_t pj[NC];  // position of the column's point in the source arrays (one dependent load, batched)
#pragma unroll
            for (int c = 0; c < NC; c++) {
              const int jl = tid + c * NT;
              ok[c] = jl < len;
              off[c] = ok[c] ? jl : 0;
              const int jj = c0 + off[c];
              pj[c] = ROWS_FAR ? ob + jj : (int64_t)POS[jj];
              raw[c] = fuse ? Vlast[jj] : 0.0;
            }
#pragma unroll
            for (int c = 0; c < NC; c++) {
              const double* cs = ROWS_FAR ? J.own.coords : J.far.coords;
              const int64_t ld = ROWS_FAR ? J.own.ld : J.far.ld;
#pragma unroll
              for (int q = 0; q < D; q++) y[c][q] = cs[q * ld + pj[c]];
            }
#pragma unroll
            for (int c = 0; c < NC; c++) {
              acc[c] = ok[c] ? kval_class<KC>(J.kind, J.a, knum, r2_exact<D>(xl, y[c])) : 0.0;  // no work on padding
              vl[c] = 0.0;
              if (fuse && ok[c]) {  // normalise row k - 1 in passing
                vl[c] = __ddiv_rn(raw[c], piv_prev);
                Vlast[c0 + off[c]] = vl[c];
                v2p += vl[c] * vl[c];
              }
            }
          }
          for (int b = 0; b < nb; b++) {
            const int r0 = b * TB;
            mbar_wait_u32(bar0 + 8u * (uint32_t)cslot, cpar);
            const double* R = ring + cslot * (TB * SEG);
            const int rows = kf - r0 < TB ? kf - r0 : TB;
#pragma unroll
            for (int g4 = 0; g4 < TB; g4 += 4) {
              if (g4 >= rows) break;  // uniform
              double p[4];
              if (g4 + 4 <= rows) {  // four whole rows: unconditional loads, then the arithmetic
                double v[4][NC];
#pragma unroll
                for (int tt = 0; tt < 4; tt++)
#pragma unroll
                  for (int c = 0; c < NC; c++) v[tt][c] = R[(g4 + tt) * SEG + off[c]];
#pragma unroll
                for (int tt = 0; tt < 4; tt++) {
                  const double ut = urow[r0 + g4 + tt];
                  p[tt] = 0.0;
#pragma unroll
                  for (int c = 0; c < NC; c++) {
                    acc[c] = __dsub_rn(acc[c], __dmul_rn(ut, v[tt][c]));
                    p[tt] = fma(v[tt][c], vl[c], p[tt]);
                  }
                }
              } else {  // last rows of the pass
#pragma unroll
                for (int tt = 0; tt < 4; tt++) {
                  p[tt] = 0.0;
                  if (g4 + tt < rows) {  // uniform
                    const double ut = urow[r0 + g4 + tt];
#pragma unroll
                    for (int c = 0; c < NC; c++) {
                      const double v = R[(g4 + tt) * SEG + off[c]];
                      acc[c] = __dsub_rn(acc[c], __dmul_rn(ut, v));
                      p[tt] = fma(v, vl[c], p[tt]);
                    }
                  }
                }
              }
              if (fuse) {
                // transpose-reduce 4 partial sums over the warp: lane gets t = r0 + g4 + ((lane >> 3) & 3)
                const bool b4 = lane & 16, b3 = lane & 8;
                double k0 = b4 ? p[2] : p[0], k1 = b4 ? p[3] : p[1];
                k0 += __shfl_xor_sync(0xffffffffu, b4 ? p[0] : p[2], 16);
                k1 += __shfl_xor_sync(0xffffffffu, b4 ? p[1] : p[3], 16);
                double kk = b3 ? k1 : k0;
                kk += __shfl_xor_sync(0xffffffffu, b3 ? k0 : k1, 8);
                kk += __shfl_xor_sync(0xffffffffu, kk, 4);
                kk += __shfl_xor_sync(0xffffffffu, kk, 2);
                kk += __shfl_xor_sync(0xffffffffu, kk, 1);
                const int tq = r0 + g4 + ((lane >> 3) & 3);
                if ((lane & 7) == 0 && tq < kf) crosspart[warp * cap + tq] += kk;
              }
            }
            __syncthreads();  // every thread is done with the slot: it takes the next batch of the stream
            if (++cslot == S) {
              cslot = 0;
              cpar ^= 1u;
            }
            inflight--;
            if (qi < Q) issue(qi++, kf, nb);
          }
          if (fuse) {
            const double ul = urow[ki - 1];
#pragma unroll
            for (int c = 0; c < NC; c++) acc[c] = __dsub_rn(acc[c], __dmul_rn(ul, vl[c]));
          }
#pragma unroll
          for (int c = 0; c < NC; c++) {
            if (ok[c]) {
              const int jj = c0 + off[c];
              Vnew[jj] = acc[c];
              if (!col_used(jj)) {
                const double val = fabs(acc[c]);
                if (val > best) {
                  best = val;
                  bj = jj;
                }
              }
            }
          }
        }
        fence_proxy_async_global();  // the rows written above are read by bulk copies (async proxy) in later passes
        APROF(1);
        if (bj < 0) best = -1.0;
        if (fuse)  // the per-warp cross partials are complete (every batch ends with a barrier): sum them
          for (int t = tid; t < kf; t += NT) {
            double w = 0.0;
            for (int q = 0; q < NW; q++) w += crosspart[q * cap + t];
            crossv[t] = w;
          }
        const double v2 = block_argmax_sum<NT>(best, bj, v2p, rs);  // its barriers also publish crossv
        // The next pass (a retry with another trial row, or step k + 1) streams rows 0 .. k - 1 whatever happens:
        // start its first batches now, so they fly during the pivot search and the column pass.  (The barriers
        // inside block_argmax order every thread's row writes + proxy fence before these copies.)
        if (ki > 0 && !(best > 0.0 && k + 1 == full)) {  // (the last step of a cell is followed by no pass)
          const int nbn = (ki + TB - 1) / TB, Qn = nseg * nbn;
          while (pre < Qn && inflight < S) issue(pre++, ki, nbn);
        }
        APROF(2);
        if (fuse) {  // finish step k - 1: norm update, stopping test
          {  // every warp forms the same sum in the same order (lanes over t, then a butterfly)
            double part = 0.0;
            for (int t = lane; t < kf; t += 32) part = fma(2.0 * crossu[t], crossv[t], part);
            norm2 += warp_sum(part);
          }
          norm2 += u2_prev * v2;
          pend = false;
          fuse = false;
          if (u2_prev * v2 <= J.eps2 * (norm2 > 0.0 ? norm2 : 0.0)) {
            stop_prev = true;
            break;
          }
        }
        nev += n;
        if (best > 0.0) break;
        int64_t first = INT64_MAX;
        for (int64_t i = tid; i < m; i += NT)
          if (!row_used((int)i) && i < first) first = i;
        first = block_min<NT>(first, rs);
        if (first == INT64_MAX) {
          exhausted = true;
          break;
        }
        trial = first;
        __syncthreads();
      }
      if (stop_prev || exhausted) break;
      if (WHICH == 0 && k + 1 == full && full == m) {
        // Last step of a cell whose rank reaches its row count (most leaves): the reference stops at k == full
        // whatever the stopping test says, every row is then a pivot row, so the interpolator is a permutation
        // and neither the last residual column nor the normalised last row is ever read.  Only the column pivot
        // found above and the evaluation count of the skipped column pass are recorded.
        if (tid == 0) {
          RP[k] = trial;
          CP[k] = bj;
        }
        nev += m;
        k += 1;
        break;
      }
      // pivot of step k; the row stays raw until the next pass normalises it
      const double piv = V[k * ldv + bj];
      if (tid < D) yb[tid] = colc(tid, bj);
      for (int64_t t = tid; t < k; t += NT) vcol[t] = V[t * ldv + bj];
      __syncthreads();
      if (tid == 0) {
        if (sbits) cbits[bj >> 5] |= 1u << (bj & 31);
        else cu[bj] = 1;
      }
      APROF(3);
      double yl[D];
#pragma unroll
      for (int q = 0; q < D; q++) yl[q] = yb[q];
      double u2p = 0.0;
      best = -1.0;  // next trial row: the largest |u| among the unused rows, found while the column is formed
      int64_t bi = -1;
      for (int64_t i = tid; i < m; i += NT) {
        double xl[D];
#pragma unroll
        for (int q = 0; q < D; q++) xl[q] = rowc(q, i);
        double acc = kval_class<KC>(J.kind, J.a, knum, r2_exact<D>(xl, yl));
        for (int64_t t = 0; t < k; t++) acc = __dsub_rn(acc, __dmul_rn(U[t * m + i], vcol[t]));
        U[k * m + i] = acc;
        u2p += acc * acc;
        if (!row_used((int)i)) {
          const double val = fabs(acc);
          if (val > best) {
            best = val;
            bi = i;
          }
        }
      }
      nev += m;
      __syncthreads();
      for (int64_t t = warp; t < k; t += NW) {
        double sacc = 0.0;
        const double* Ut = U + t * m;
        const double* Uk = U + k * m;
        for (int64_t i = lane; i < m; i += 32) sacc += Ut[i] * Uk[i];
        sacc = warp_sum(sacc);
        if (lane == 0) crossu[t] = sacc;
      }
      APROF(5);
      const double u2 = block_argmax_sum<NT>(best, bi, u2p, rs);  // syncs: crossu visible
      if (tid == 0) {
        RP[k] = trial;
        CP[k] = bj;
      }
      piv_prev = piv;
      u2_prev = u2;
      k += 1;
      if (k == full) {  // the reference stops here whatever its eps test says (converged stays true)
        finish_row((int)k - 1, false);
        break;
      }
      if (k == cap) {  // eps test decides between converged and not
        const double v2 = finish_row((int)k - 1, true);
        for (int64_t t = 0; t < k - 1; t++) norm2 += 2.0 * crossu[t] * crossv[t];
        norm2 += u2 * v2;
        if (!(u2 * v2 <= J.eps2 * (norm2 > 0.0 ? norm2 : 0.0))) converged = 0;
        break;
      }
      APROF(6);
      if (bi < 0) {  // the reference breaks after its (here irrelevant) stopping test
        finish_row((int)k - 1, false);
        break;
      }
      trial = bi;
      pend = true;
      __syncthreads();
    }
    // batches prefetched for a pass that never came: consume them so the ring and the parities stay in step
    for (; pre > 0; pre--) {
      mbar_wait_u32(bar0 + 8u * (uint32_t)cslot, cpar);
      if (++cslot == S) {
        cslot = 0;
        cpar ^= 1u;
      }
      inflight--;
    }
    __syncthreads();
    APROF(6);
    const int64_t po = J.piv_off[cell];
    if (tid == 0) {
      J.rank[cell] = k;
      J.conv[cell] = converged;
      J.nevals[cell] = nev;
    }
    for (int64_t t = tid; t < k; t += NT) {
      const int64_t r = RP[t], c = CP[t];
      J.tpiv[po + t] = ROWS_FAR ? J.far.gidx[POS[r]] : J.own.gidx[ob + r];
      J.spiv[po + t] = ROWS_FAR ? J.own.gidx[ob + c] : J.far.gidx[POS[c]];
    }
    // interpolation operator (aca.py:297 / :311, same arithmetic): which 0 -> P = U L^{-1}; 1 -> Q = V R^{-T}.
    // The back substitution re-reads the columns of P it has already formed: when the operator fits, it is built
    // in the (now idle) ring and copied out coalesced.
    if (k > 0) {
      const int64_t rows = WHICH == 0 ? m : n;
      const int64_t fs = WHICH == 0 ? m : ldv;  // row stride of the factor
      const double* F = WHICH == 0 ? U : V;
      const int64_t* pv = WHICH == 0 ? RP : CP;
      double* Pg = J.mat + J.mat_off[cell];
      const bool staged = k * rows <= (int64_t)S * TB * SEG;
      double* P = staged ? ring : Pg;
      // a full-rank cell (every row is a pivot row: most leaves) needs no back substitution: the pinning below
      // overwrites every row with its unit row, exactly what the reference's interpolator ends up as
      if (k < rows)
        for (int64_t i = tid; i < rows; i += NT) {
          for (int64_t sI = k - 1; sI >= 0; sI--) {
            const double* Fs = F + sI * fs;
            double acc = Fs[i];
            for (int64_t t = sI + 1; t < k; t++) acc -= P[t * rows + i] * Fs[pv[t]];
            P[sI * rows + i] = WHICH == 0 ? acc / Fs[pv[sI]] : acc;
          }
        }
      __syncthreads();
      {
        const int ki = (int)k;
        for (int q = tid; q < ki * ki; q += NT) {
          const int t = q / ki, sI = q - t * ki;
          P[(int64_t)sI * rows + pv[t]] = (sI == t) ? 1.0 : 0.0;
        }
      }
      if (staged) {
        __syncthreads();
        for (int64_t q = tid; q < k * rows; q += NT) Pg[q] = P[q];
        fence_proxy_async();  // generic writes to the ring before the next cell's bulk copies into it
      }
    }
    APROF(7);
  }
}

template <int D, int NT>
void set_aca_smem(size_t bytes) {
  // the attribute is per device: set on every call that needs the opt-in (a process may drive several GPUs)
  if (bytes > 40 * 1024)
    CK(cudaFuncSetAttribute(aca_kernel<D, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// One side (incoming or outgoing) of the NNCA for one level.
//   rows/cols: either "own" (contiguous range of a source) or "far"
//   (gathered concatenation over the interaction list).
struct SideResult {
  std::vector<int64_t> rank_h;
  DBuf<int64_t> rank, tpiv, spiv, piv_off, conv, nevals;
  DBuf<double> mat;  // interpolation operator per cell (col-major)
  DBuf<int64_t> mat_off, mat_rows;
};

// Per-device ACA workspace arena: grows to the largest launch seen and is reused after that, so repeated setups
// do not map memory again (mapping ~100 GB for c1's top levels costs 650 ms).  It is a plain cudaMalloc block,
// outside the stream-ordered pool: its size is budgeted against the device's free memory, and memory the pool
// holds (reserved or cached) is not available to it, so the budget can never over-commit.  Assemblies on one
// device are serialised by the arena's mutex (each one fills the GPU anyway); h2b_release_workspace() frees the
// arenas (they are deliberately not freed at process exit).
struct DeviceArena {
  std::mutex mu;
  double* p = nullptr;
  size_t n = 0;  // doubles
};
DeviceArena* device_arenas() {
  static DeviceArena* arenas = new DeviceArena[64];
  return arenas;
}
DeviceArena& current_arena() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  return device_arenas()[dev & 63];
}
double* aca_arena(DeviceArena& A, size_t doubles, cudaStream_t s) {
  if (A.n < doubles) {
    CK(cudaStreamSynchronize(s));
    if (A.p) CK(cudaFree(A.p));
    A.p = nullptr;
    A.n = 0;
    const size_t want = doubles + doubles / 8;
    if (cudaMalloc(reinterpret_cast<void**>(&A.p), want * sizeof(double)) == cudaSuccess) {
      A.n = want;
    } else {
      cudaGetLastError();  // the head room was a bonus: take exactly what the launch needs
      CK(cudaMalloc(reinterpret_cast<void**>(&A.p), doubles * sizeof(double)));
      A.n = doubles;
    }
  }
  return A.p;
}

// ring configurations: threads per CTA, columns per thread, rows per batch, CTAs per SM
template <int D, int KC, int NT, int NC, int TB, int MB, bool OUT>
struct RingCfg {
  static constexpr int nt = NT, seg = NT * NC, slot = TB * NT * NC, mb = MB;  // slot: doubles per ring slot
  static auto kern() { return aca_ring<D, KC, NT, NC, TB, MB, OUT>; }
};

template <int D, int KC>
void run_side(const DevTree& T, int level, bool rows_far, const Src& own, const Src& far, int kind, double a,
              double eps, int64_t max_rank, int which_interp, SideResult& R, DeviceArena& arena, cudaStream_t s) {
  const auto wall0 = std::chrono::steady_clock::now();
  const DevLevel& L = T.lv[level];
  const int64_t n = L.n;
  DBuf<int64_t> own_b, own_len, far_len;
  own_b.alloc(std::max<int64_t>(n, 1));
  own_len.alloc(std::max<int64_t>(n, 1));
  far_len.alloc(std::max<int64_t>(n, 1));
  if (n)
    cand_sizes<<<ceil_div(n, 128), 128, 0, s>>>(n, own, far, L.il_ptr.get(), L.il_idx.get(), own_b.get(),
                                                own_len.get(), far_len.get());
  CKL();
  auto ol = to_host(own_len.get(), n, s), fl = to_host(far_len.get(), n, s);
  const auto wall1 = std::chrono::steady_clock::now();
  std::vector<int64_t> mh(n), nh(n), caph(n), piv_off(n), mat_off(n), order(n);
  int64_t m_max = 1, n_max = 1, f_max = 1, cap_max = 1;
  for (int64_t c = 0; c < n; c++) {
    mh[c] = rows_far ? fl[c] : ol[c];
    nh[c] = rows_far ? ol[c] : fl[c];
    int64_t cp = std::min(mh[c], nh[c]);
    if (max_rank >= 0) cp = std::min(cp, max_rank);
    caph[c] = cp;
    m_max = std::max(m_max, mh[c]);
    n_max = std::max(n_max, nh[c]);
    f_max = std::max(f_max, fl[c]);
    cap_max = std::max(cap_max, cp);
  }
  int64_t po = 0, mo = 0;
  for (int64_t c = 0; c < n; c++) {
    piv_off[c] = po;
    po += caph[c];
    mat_off[c] = mo;
    mo += (which_interp == 0 ? mh[c] : nh[c]) * caph[c];
  }
  {  // work order: largest (m + n) * cap first, ties by cell index (two-pass LSD radix sort, 16-bit digits;
     // std::stable_sort took ~5 ms of host time per setup at the 70K-cell leaf level)
    std::vector<int64_t> key(n);
    int64_t kmax = 0;
    for (int64_t c = 0; c < n; c++) {
      key[c] = (mh[c] + nh[c]) * caph[c];
      kmax = std::max(kmax, key[c]);
      order[c] = c;
    }
    if (kmax >= (int64_t(1) << 32)) {
      std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) { return key[x] > key[y]; });
    } else {
      std::vector<int64_t> tmp(n);
      std::vector<int64_t> cnt(65537);
      for (int sh = 0; sh < 32 && (sh == 0 || (kmax >> sh) != 0); sh += 16) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t i = 0; i < n; i++) cnt[((kmax - key[order[i]]) >> sh & 0xFFFF) + 1]++;
        for (int dg = 0; dg < 65536; dg++) cnt[dg + 1] += cnt[dg];
        for (int64_t i = 0; i < n; i++) tmp[cnt[(kmax - key[order[i]]) >> sh & 0xFFFF]++] = order[i];
        order.swap(tmp);
      }
    }
  }
  const auto wall1b = std::chrono::steady_clock::now();
  R.piv_off = upload(piv_off, s);
  R.rank.alloc(std::max<int64_t>(n, 1));
  R.conv.alloc(std::max<int64_t>(n, 1));
  R.nevals.alloc(std::max<int64_t>(n, 1));
  R.tpiv.alloc(std::max<int64_t>(po, 1));
  R.spiv.alloc(std::max<int64_t>(po, 1));
  R.mat_off = upload(mat_off, s);
  R.mat_rows = upload(which_interp == 0 ? mh : nh, s);
  R.mat.alloc(std::max<int64_t>(mo, 1));
  if (n == 0) {
    R.rank_h.clear();
    return;
  }
  if (far.ld >= ((int64_t)1 << 31) || own.ld >= ((int64_t)1 << 31) || f_max >= ((int64_t)1 << 31))
    throw std::invalid_argument("more than 2^31 candidate positions in an NNCA level");
  auto d_cap = upload(caph, s);
  auto d_order = upload(order, s);
  int dev = 0, nsm = 0, smem_sm = 0, smem_cta = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  CK(cudaDeviceGetAttribute(&smem_cta, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const auto wall2 = std::chrono::steady_clock::now();
  if (getenv("H2B_SETUP_VERBOSE"))
    fprintf(stderr, "[h2b] level %d side %d: host prep = vectors + sort %.3f ms, allocations + uploads %.3f ms\n", level,
            which_interp, std::chrono::duration<double, std::milli>(wall1b - wall1).count(),
            std::chrono::duration<double, std::milli>(wall2 - wall1b).count());
  CellJob J;
  J.kind = kind;
  J.a = a;
  J.eps2 = eps * eps;
  J.rows_far = rows_far ? 1 : 0;
  J.own = own;
  J.far = far;
  J.il_ptr = L.il_ptr.get();
  J.il_idx = L.il_idx.get();
  J.caps = d_cap.get();
  J.piv_off = R.piv_off.get();
  J.tpiv = R.tpiv.get();
  J.spiv = R.spiv.get();
  J.rank = R.rank.get();
  J.conv = R.conv.get();
  J.nevals = R.nevals.get();
  J.mat = R.mat.get();
  J.mat_off = R.mat_off.get();
  J.which = which_interp;
  J.f_max = f_max;
  J.cap_max = cap_max;
  J.ncell = n;
  J.order = d_order.get();
  static const bool verbose = getenv("H2B_SETUP_VERBOSE") != nullptr;
  auto launch = [&](auto cfg) -> bool {  // false: the rank cap does not fit this configuration's shared memory
    using C = decltype(cfg);
    auto kern = C::kern();
    // shared memory: 4 cap-sized vectors and the per-warp cross partials, then as many ring slots as fit (deep
    // prefetch hides the DRAM latency of the residual rows), then U for the cells whose cap x m fits in the rest
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));  // static shared memory; every CTA also reserves 1 KB
    int64_t bit_words = (((m_max + 31) >> 5) + ((n_max + 31) >> 5) + 3) & ~(int64_t)1;
    if (bit_words > aca_bit_words(C::nt)) bit_words = 0;  // very long candidate lists keep byte flags in the slab
    J.bit_words = (int)bit_words;
    const int64_t vecs = (4 + C::nt / 32) * cap_max;
    int64_t u_need = 0;
    for (int64_t c = 0; c < n; c++) u_need = std::max(u_need, caph[c] * mh[c]);
    const int64_t u_pref = std::min<int64_t>(u_need, H2B_ACA_UPREF);
    // this CTA's share of the SM at C::mb CTAs per SM; fewer CTAs per SM when two ring slots do not fit in it
    int64_t share = 0, slots = 0;
    for (int mb = C::mb; mb >= 1 && slots < 2; mb--) {
      share = (std::min<int64_t>(smem_cta, smem_sm / mb - 1024) - (int64_t)fa.sharedSizeBytes) / 8 - 16;
      slots = (share - vecs - u_pref) / C::slot;
      if (slots < 2) slots = (share - vecs) / C::slot;
    }
    if (slots < 2) return false;
    slots = std::min<int64_t>(slots, H2B_ACA_SLOTS);
    J.slots = (int)slots;
    const int64_t fixed = slots * C::slot + vecs;
    J.u_smem = std::max<int64_t>(0, std::min<int64_t>(u_need, share - fixed));
    const size_t smem = (size_t)(fixed + J.u_smem) * sizeof(double);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, C::nt, smem));
    int64_t grid = std::min<int64_t>(n, (int64_t)nsm * std::max(per, 1));
    int64_t us = 0, vs = 0;
    for (int64_t c = 0; c < n; c++) {
      if (caph[c] * mh[c] > J.u_smem) us = std::max(us, caph[c] * mh[c]);
      vs = std::max(vs, (caph[c] + 1) * ((nh[c] + 1) & ~(int64_t)1));  // + 1: the speculative last row pass
    }
    J.u_slab = (us + 1) & ~(int64_t)1;
    J.v_slab = vs;
    int64_t ws = J.u_slab + J.v_slab + (f_max + 1) / 2 + 2 * cap_max + (m_max + n_max + 7) / 8 + 1;
    ws = (ws + 31) / 32 * 32 + H2B_ACA_SLAB_PAD;  // pad: per-CTA slabs off power-of-two strides
    if (grid * ws > (int64_t)arena.n) {
      // Slabs are sized for the rank cap (min(m, n)): the top levels of dense clouds (n ~ 1e5 candidates per
      // cell) need ~0.8 GB per concurrent cell, so their total is bounded by the device's free memory plus what
      // the arena already holds -- fewer concurrent cells instead of running out.  An arena that already holds
      // >= 3/4 of the wanted slabs is used as is: growing it means mapping tens of GB again for a <= 25% longer
      // launch.  Steady-state setups skip the query.
      const int64_t have = (int64_t)arena.n / ws;
      if (have >= 1 && 4 * have >= 3 * grid) {
        grid = have;
      } else {
        size_t fr = 0, tot = 0;
        CK(cudaMemGetInfo(&fr, &tot));
        const int64_t budget = (int64_t)(0.6 * (double)fr / sizeof(double)) + (int64_t)arena.n;
        grid = std::max<int64_t>(1, std::min<int64_t>(grid, budget / ws));
      }
    }
    double* wsbuf = aca_arena(arena, (size_t)(grid * ws), s);
    DBuf<unsigned long long> counter;
    counter.alloc(1);
    CK(cudaMemsetAsync(counter.get(), 0, sizeof(unsigned long long), s));
    J.ws = wsbuf;
    J.ws_doubles = ws;
    J.counter = counter.get();
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (verbose) {
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, s));
    }
    kern<<<(unsigned)grid, C::nt, smem, s>>>(J);
    CKL();
    if (verbose) {
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      fprintf(stderr,
              "[h2b] level %d side %d: %lld cells, m_max %lld n_max %lld cap_max %lld, grid %lld x %d (%d per SM), "
              "segment %d x %d slots, smem %zu B (U %lld doubles): %.3f ms\n",
              level, which_interp, (long long)n, (long long)m_max, (long long)n_max, (long long)cap_max,
              (long long)grid, C::nt, per, C::seg, J.slots, smem, (long long)J.u_smem, ms);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
#ifdef H2B_ACA_PROF
      unsigned long long pr[8];
      CK(cudaMemcpyFromSymbol(pr, g_aca_prof, sizeof pr));
      fprintf(stderr, "[h2b]   phase cycles (sum over CTAs, 1e6): gather %.1f row %.1f argmax %.1f norm %.1f cross %.1f col %.1f "
              "tail %.1f interp %.1f\n", pr[0] / 1e6, pr[1] / 1e6, pr[2] / 1e6, pr[3] / 1e6, pr[4] / 1e6, pr[5] / 1e6,
              pr[6] / 1e6, pr[7] / 1e6);
      unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      CK(cudaMemcpyToSymbol(g_aca_prof, z, sizeof z));
#endif
    }
    return true;
  };
  // Many cells: small CTAs, several per SM (independent cells hide each other's barriers and latencies); few
  // cells (upper levels): wide CTAs so one cell's row pass uses the whole SM.
  // The per-warp vectors scale with the rank cap: a cap too large for the preferred configuration falls back to
  // the narrower ones (fewer warps, smaller ring slots).
  auto small = [&] {
    return rows_far ? launch(RingCfg<D, KC, H2B_ACA_NT_S, H2B_ACA_NC_S, H2B_ACA_TB_S, H2B_ACA_MB_S, true>{})
                    : launch(RingCfg<D, KC, H2B_ACA_NT_S, H2B_ACA_NC_S, H2B_ACA_TB_S, H2B_ACA_MB_S, false>{});
  };
  auto mid = [&] {
    return rows_far ? launch(RingCfg<D, KC, 256, 4, 4, 2, true>{}) : launch(RingCfg<D, KC, 256, 4, 4, 2, false>{});
  };
  auto wide = [&] {
    return rows_far ? launch(RingCfg<D, KC, H2B_ACA_NT, H2B_ACA_NC, H2B_ACA_TB, H2B_ACA_MINB, true>{})
                    : launch(RingCfg<D, KC, H2B_ACA_NT, H2B_ACA_NC, H2B_ACA_TB, H2B_ACA_MINB, false>{});
  };
  bool done;
  if (n >= H2B_ACA_CELLS_S) done = small();
  else if (n >= H2B_ACA_CELLS_M) done = mid() || small();
  else done = wide() || mid() || small();
  if (!done) throw std::runtime_error("ACA rank cap too large for shared memory");
  CK(cudaStreamSynchronize(s));
  const auto wall3 = std::chrono::steady_clock::now();
  R.rank_h = to_host(R.rank.get(), n, s);
  if (verbose) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[h2b] level %d side %d: run_side wall %.3f ms (sizes %.3f, host prep %.3f, ACA %.3f, tail %.3f)\n",
            level, which_interp, ms(wall0, std::chrono::steady_clock::now()), ms(wall0, wall1), ms(wall1, wall2),
            ms(wall2, wall3), ms(wall3, std::chrono::steady_clock::now()));
  }
}
template <int D, int KC>
std::unique_ptr<DevH2> assemble_impl(const DevTree& T, int kind, double a, double eps, bool force_general,
                                     int64_t max_rank, cudaStream_t s) {
  DeviceArena& arena = current_arena();
  std::lock_guard<std::mutex> arena_lock(arena.mu);  // one assembly per device at a time (shared workspace)
  auto t0 = std::chrono::steady_clock::now();
  auto H = std::make_unique<DevH2>();
  H->t = &T;
  H->kind = kind;
  H->a = a;
  H->eps = eps;
  H->symmetric = T.shared && !force_general;  // all built-in kernels are symmetric
  const int L = T.depth;
  H->lv.resize(L + 1);
  std::vector<std::vector<int64_t>> kin_h(L + 1);
  for (int level = L; level >= 2; level--) {
    const DevLevel& Lv = T.lv[level];
    DevH2Level& HL = H->lv[level];
    HL.n = Lv.n;
    const bool leaf = level == L;
    Src own_t, own_s, far_t, far_s;
    if (leaf) {
      own_t = Src{T.tsd(), T.np, T.t_perm.get(), Lv.t_ptr.get(), nullptr};
      own_s = Src{T.ssd(), T.nq, T.sperm(), T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get(), nullptr};
    } else {
      const DevH2Level& C = H->lv[level + 1];
      own_t = Src{C.tin_c.get(), std::max<int64_t>(C.in_total, 1), C.t_in.get(), C.in_ptr.get(), Lv.ch_ptr.get()};
      own_s = Src{C.sout_cd(), std::max<int64_t>(C.out_total, 1), C.s_out.n ? C.s_out.get() : C.t_in.get(),
                  C.out_ptrd(), Lv.ch_ptr.get()};
    }
    far_t = own_t;
    far_s = own_s;
    // incoming: rows = own targets, cols = far sources
    SideResult in;
    run_side<D, KC>(T, level, false, own_t, far_s, kind, a, eps, max_rank, 0, in, arena, s);
    HL.kin = std::move(in.rank);
    {  // pivot offsets from the ranks already on the host (no device scan + read-back)
      std::vector<int64_t> ptr(HL.n + 1, 0);
      for (int64_t c = 0; c < HL.n; c++) ptr[c + 1] = ptr[c] + in.rank_h[c];
      HL.in_total = ptr[HL.n];
      HL.in_ptr = upload(ptr, s, &H->mem);
      kin_h[level] = std::move(in.rank_h);
    }
    HL.t_in.alloc(std::max<int64_t>(HL.in_total, 1), &H->mem);
    HL.s_in.alloc(std::max<int64_t>(HL.in_total, 1), &H->mem);
    if (HL.n)
      compact_pivots<<<(unsigned)HL.n, 64, 0, s>>>(HL.n, HL.kin.get(), in.piv_off.get(), HL.in_ptr.get(),
                                                  in.tpiv.get(), in.spiv.get(), HL.t_in.get(), HL.s_in.get());
    CKL();
    HL.tin_c.alloc(std::max<int64_t>(HL.in_total * D, 1), &H->mem);
    if (HL.in_total)
      gather_coords<D><<<ceil_div(HL.in_total, 256), 256, 0, s>>>(T.Pd(), HL.t_in.get(), HL.in_total,
                                                                  HL.tin_c.get());
    CKL();
    HL.pmat = std::move(in.mat);
    HL.pm_off = std::move(in.mat_off);
    HL.m_in = std::move(in.mat_rows);
    HL.conv = std::move(in.conv);
    HL.nevals = std::move(in.nevals);
    if (!H->symmetric) {
      // outgoing: rows = far targets, cols = own sources
      SideResult out;
      run_side<D, KC>(T, level, true, own_s, far_t, kind, a, eps, max_rank, 1, out, arena, s);
      HL.kout = std::move(out.rank);
      HL.out_ptr.alloc(HL.n + 1, &H->mem);
      excl_scan(HL.kout.get(), HL.n, HL.out_ptr.get(), s);
      HL.out_total = read_one(HL.out_ptr.get() + HL.n, s);
      HL.t_out.alloc(std::max<int64_t>(HL.out_total, 1), &H->mem);
      HL.s_out.alloc(std::max<int64_t>(HL.out_total, 1), &H->mem);
      if (HL.n)
        compact_pivots<<<(unsigned)HL.n, 64, 0, s>>>(HL.n, HL.kout.get(), out.piv_off.get(), HL.out_ptr.get(),
                                                    out.tpiv.get(), out.spiv.get(), HL.t_out.get(), HL.s_out.get());
      CKL();
      HL.sout_c.alloc(std::max<int64_t>(HL.out_total * D, 1), &H->mem);
      if (HL.out_total)
        gather_coords<D><<<ceil_div(HL.out_total, 256), 256, 0, s>>>(T.Qd(), HL.s_out.get(), HL.out_total,
                                                                     HL.sout_c.get());
      CKL();
      HL.qmat = std::move(out.mat);
      HL.qm_off = std::move(out.mat_off);
      HL.n_out = std::move(out.mat_rows);
      // nevals: add outgoing counts
      auto a1 = to_host(HL.nevals.get(), HL.n, s), a2 = to_host(out.nevals.get(), HL.n, s);
      for (int64_t c = 0; c < HL.n; c++) a1[c] += a2[c];
      CK(cudaMemcpyAsync(HL.nevals.get(), a1.data(), HL.n * 8, cudaMemcpyHostToDevice, s));
      auto cv = to_host(out.conv.get(), HL.n, s);
      for (int64_t c = 0; c < HL.n; c++) H->unconverged += cv[c] == 0;
    } else {
      HL.out_total = HL.in_total;
    }
    H->cells_visited += HL.n;
  }
  // stats: one batch of read-backs after all levels
  {
    std::vector<std::vector<int64_t>> nev(L + 1), kout(L + 1), cv(L + 1);
    for (int level = 2; level <= L; level++) {
      const DevH2Level& HL = H->lv[level];
      nev[level].resize(HL.n);
      cv[level].resize(HL.n);
      if (!HL.n) continue;
      CK(cudaMemcpyAsync(nev[level].data(), HL.nevals.get(), HL.n * 8, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(cv[level].data(), HL.conv.get(), HL.n * 8, cudaMemcpyDeviceToHost, s));
      if (!H->symmetric) {
        kout[level].resize(HL.n);
        CK(cudaMemcpyAsync(kout[level].data(), HL.kout.get(), HL.n * 8, cudaMemcpyDeviceToHost, s));
      }
    }
    CK(cudaStreamSynchronize(s));
    for (int level = 2; level <= L; level++)
      for (int64_t c = 0; c < H->lv[level].n; c++) {
        H->evals_pivots += nev[level][c];
        H->max_rank = std::max(H->max_rank, kin_h[level][c]);
        if (!H->symmetric) H->max_rank = std::max(H->max_rank, kout[level][c]);
        H->unconverged += cv[level][c] == 0;
      }
  }
  static const bool verbose = getenv("H2B_SETUP_VERBOSE") != nullptr;
  auto stamp = [&](const char* what) {
    if (verbose)
      fprintf(stderr, "[h2b] assemble %s at %.3f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  stamp("levels done");
  // coupling / near-field entry counts (what the reference would evaluate)
  {
    DBuf<unsigned long long> acc;
    acc.alloc(1);
    CK(cudaMemsetAsync(acc.get(), 0, 8, s));
    for (int level = 2; level <= L; level++) {
      const DevLevel& Lv = T.lv[level];
      const DevH2Level& HL = H->lv[level];
      if (Lv.n)
        coupling_counts<<<ceil_div(Lv.n, 128), 128, 0, s>>>(Lv.n, HL.kin.get(), HL.koutd(), Lv.il_ptr.get(),
                                                            Lv.il_idx.get(), acc.get());
      CKL();
    }
    H->evals_couplings = (int64_t)read_one(acc.get(), s);
    CK(cudaMemsetAsync(acc.get(), 0, 8, s));
    const DevLevel& Lf = T.lv[L];
    near_counts<<<ceil_div(Lf.n, 128), 128, 0, s>>>(Lf.n, Lf.t_ptr.get(),
                                                    T.shared ? Lf.t_ptr.get() : Lf.s_ptr.get(), Lf.nb_ptr.get(),
                                                    Lf.nb_idx.get(), acc.get());
    CKL();
    H->evals_nearfield = (int64_t)read_one(acc.get(), s);
  }
  stamp("counts done");
  prepare_matvec(*H, s);  // interaction work list + scratch are part of the setup
  CK(cudaStreamSynchronize(s));
  stamp("matvec prepared");
  H->setup_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  return H;
}

}  // namespace

std::unique_ptr<DevH2> assemble(const DevTree& t, int kind, double a, double eps, bool force_general,
                                int64_t max_rank, cudaStream_t s) {
  if (!(eps > 0)) throw std::invalid_argument("epsilon must be positive");
  if (!kind_valid(kind)) throw std::invalid_argument("unknown kernel kind");
#define H2B_ASM(D)                                                                              \
  switch (kind_class(kind)) {                                                                   \
    case KC_INV: return assemble_impl<D, KC_INV>(t, kind, a, eps, force_general, max_rank, s); \
    case KC_EXP: return assemble_impl<D, KC_EXP>(t, kind, a, eps, force_general, max_rank, s); \
    default: return assemble_impl<D, KC_LOG>(t, kind, a, eps, force_general, max_rank, s);     \
  }
  switch (t.d) {
    case 1: H2B_ASM(1)
    case 2: H2B_ASM(2)
    case 3: H2B_ASM(3)
    default: H2B_ASM(4)
  }
#undef H2B_ASM
}

void release_workspace() {
  int cur = 0, ndev = 0;
  if (cudaGetDevice(&cur) != cudaSuccess || cudaGetDeviceCount(&ndev) != cudaSuccess) return;
  for (int dv = 0; dv < ndev && dv < 64; dv++) {
    DeviceArena& A = device_arenas()[dv];
    std::lock_guard<std::mutex> g(A.mu);
    if (!A.p) continue;
    CK(cudaSetDevice(dv));
    CK(cudaDeviceSynchronize());
    CK(cudaFree(A.p));
    A.p = nullptr;
    A.n = 0;
  }
  CK(cudaSetDevice(cur));
}

// Single-block ACA for the drop-in partial_aca path (_core.pyx:70).
void aca_single(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d, double eps,
                int64_t cap, double* U, double* V, int64_t* rp, int64_t* cp, int* conv, int64_t* nevals,
                int64_t* rank) {
  cudaStream_t s = 0;
  if (m == 0 || n == 0 || cap == 0) {
    *rank = 0;
    *conv = (m == 0 || n == 0) ? 1 : 0;
    *nevals = 0;
    return;
  }
  std::vector<double> xs(m * d), ys(n * d);
  for (int64_t i = 0; i < m; i++)
    for (int k = 0; k < d; k++) xs[k * m + i] = X[i * d + k];
  for (int64_t j = 0; j < n; j++)
    for (int k = 0; k < d; k++) ys[k * n + j] = Y[j * d + k];
  auto dx = upload(xs, s), dy = upload(ys, s);
  std::vector<int64_t> z{0}, mh{m}, nh{n}, ch{cap}, fo{0};
  auto dz = upload(z, s), dm = upload(mh, s), dn = upload(nh, s), dc = upload(ch, s);
  DBuf<double> dU, dV;
  DBuf<unsigned char> fl;
  DBuf<int64_t> drp, dcp, tp, sp, rk, cv, ne;
  dU.alloc(m * cap);
  dV.alloc(n * cap);
  fl.alloc(m + n);
  drp.alloc(cap);
  dcp.alloc(cap);
  tp.alloc(cap);
  sp.alloc(cap);
  rk.alloc(1);
  cv.alloc(1);
  ne.alloc(1);
  AcaArgs A;
  A.kind = kind;
  A.a = a;
  A.eps2 = eps * eps;
  A.cell0 = 0;
  A.m = dm.get();
  A.n = dn.get();
  A.cap = dc.get();
  A.row_base = dx.get();
  A.ld_row = m;
  A.row_off = dz.get();
  A.row_gidx = nullptr;
  A.col_base = dy.get();
  A.ld_col = n;
  A.col_off = dz.get();
  A.col_gidx = nullptr;
  A.U = dU.get();
  A.u_off = dz.get();
  A.V = dV.get();
  A.v_off = dz.get();
  A.flags = fl.get();
  A.f_off = dz.get();
  A.piv_off = dz.get();
  A.rp = drp.get();
  A.cp = dcp.get();
  A.tpiv = tp.get();
  A.spiv = sp.get();
  A.rank = rk.get();
  A.conv = cv.get();
  A.nevals = ne.get();
  size_t smem = (size_t)cap * 4 * sizeof(double);
  if (smem > 200 * 1024) throw std::runtime_error("ACA rank cap too large for shared memory");
  switch (d) {
    case 1: set_aca_smem<1, 256>(smem); aca_kernel<1, 256><<<1, 256, smem, s>>>(A); break;
    case 2: set_aca_smem<2, 256>(smem); aca_kernel<2, 256><<<1, 256, smem, s>>>(A); break;
    case 3: set_aca_smem<3, 256>(smem); aca_kernel<3, 256><<<1, 256, smem, s>>>(A); break;
    default: set_aca_smem<4, 256>(smem); aca_kernel<4, 256><<<1, 256, smem, s>>>(A); break;
  }
  CKL();
  int64_t k = read_one(rk.get(), s);
  *rank = k;
  *conv = (int)read_one(cv.get(), s);
  *nevals = read_one(ne.get(), s);
  auto hU = to_host(dU.get(), m * cap, s), hV = to_host(dV.get(), n * cap, s);
  auto hr = to_host(drp.get(), cap, s), hc = to_host(dcp.get(), cap, s);
  for (int64_t i = 0; i < m; i++)
    for (int64_t t = 0; t < k; t++) U[i * cap + t] = hU[t * m + i];
  for (int64_t j = 0; j < n; j++)
    for (int64_t t = 0; t < k; t++) V[j * cap + t] = hV[t * n + j];
  for (int64_t t = 0; t < k; t++) {
    rp[t] = hr[t];
    cp[t] = hc[t];
  }
}

}  // namespace h2b
