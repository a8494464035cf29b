// interact.cuh — the FP64 interaction kernel shared by the per-dimension
// translation units interact_d{1,2,3,4}.cu (split so nvcc compiles the
// D x kernel-kind x RHS-width instantiations in parallel).
#pragma once
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"

namespace h2b {

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


// ---------------------------------------------------------------------
// Interaction kernel: one launch for every M2L level and the near field.
//
// Work item = (list, cell): list l in [2, L] is level l's interaction list
// (targets = the cell's incoming pivots, sources = the outgoing pivots of its
// interaction-list cells with their multipole charges); list L + 1 is the
// leaf near field (points, input charges).  Items are sorted by pair count,
// largest first, so all levels share one balanced grid.  A CTA owns one
// target cell: 2 targets per thread in registers, the source list streamed
// through a shared-memory tile (coordinates + charges, LDS.128 broadcasts).
// ---------------------------------------------------------------------
namespace {

#ifndef H2B_IT2
#define H2B_IT2 128
#endif
#ifndef H2B_TILE1
#define H2B_TILE1 512
#endif
constexpr int IT2 = H2B_IT2;
constexpr int MAXMEM = IT2;

struct LevelTab {
  const double* tc;      // target coords SoA (ld_t)
  int64_t ld_t;
  const int64_t* t_ptr;  // target range per cell
  const double* sc;      // source coords SoA (ld_s)
  int64_t ld_s;
  const int64_t* s_ptr;  // source range per source cell
  const double* q;       // charges, row stride R
  const int64_t* l_ptr;  // cell list (CSR)
  const int64_t* l_idx;
  double* out;           // result rows (target position) * R
};

__device__ __forceinline__ double rsq_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// K(r2) for the interaction kernel.  1/r: MUFU.RSQ64H seed + one Newton step
// (cubic correction: ~1 ulp), with the punctured diagonal handled by
// an integer test on the high word (r2 == 0 or subnormal -> 0).
template <int KIND>
__device__ __forceinline__ double kpair(double r2, const KParams& kp) {
  if constexpr (KIND == COULOMB || KIND == LAPLACE) {
    const bool zero = __double2hiint(r2) == 0;
    const double r2s = zero ? 1.0 : r2;
    const double y = rsq_approx(r2s);
    const double e = fma(-r2s, y * y, 1.0);
    const double kv = fma(y * e, fma(0.375, e, 0.5), y);  // y (1 + e/2 + 3e^2/8): full FP64 accuracy
    return zero ? 0.0 : kv;
  } else {
    return kfast<KIND>(r2, kp);
  }
}

// Per-source record in shared memory: D coordinates then NR charges, padded
// to whole double2 words so one source is W LDS.128 broadcasts.
template <int D, int NR>
struct SrcW {
  static constexpr int W = (D + NR + 1) / 2;
};

// Body for one target chunk.  RT = 2 targets per thread (register blocking:
// every shared-memory source read feeds two pair evaluations).  SELF = the
// list may contain the target itself (near field): punctured diagonal test.
template <int D, int KIND, int NR, int TILE, bool SELF, int RT>
__device__ __forceinline__ void interact_cell(const LevelTab& T, int64_t c, int64_t R, int64_t r0, const KParams& kp,
                                              double2* tile, int64_t* pref, int64_t* sbeg, int64_t* wsum,
                                              double* part) {
  constexpr int W = SrcW<D, NR>::W;
  const int64_t tb = T.t_ptr[c], m = T.t_ptr[c + 1] - tb;
  const int64_t lb = T.l_ptr[c], le = T.l_ptr[c + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t a0 = 0; a0 < m; a0 += RT * IT2) {
    const int64_t mc = (m - a0) < RT * IT2 ? (m - a0) : RT * IT2;
    const int TS = (int)((mc + RT - 1) / RT);
    const int G = IT2 / TS;
    const int slot = tid % TS, grp = tid / TS;
    const bool worker = grp < G;
    bool act[RT];
    double x[RT][D];
    double acc[RT][NR];
#pragma unroll
    for (int t = 0; t < RT; t++) {
      const int64_t a = a0 + slot + t * TS;
      act[t] = worker && (slot + t * TS) < mc;
#pragma unroll
      for (int k = 0; k < D; k++) x[t][k] = act[t] ? T.tc[k * T.ld_t + tb + a] : 0.0;
#pragma unroll
      for (int r = 0; r < NR; r++) acc[t][r] = 0.0;
    }
    for (int64_t q0 = lb; q0 < le; q0 += MAXMEM) {
      const int nmem = (int)(le - q0 < MAXMEM ? le - q0 : MAXMEM);
      int64_t len = 0;
      if (tid < nmem) {
        const int64_t sc = T.l_idx[q0 + tid];
        const int64_t b = T.s_ptr[sc];
        sbeg[tid] = b;
        len = T.s_ptr[sc + 1] - b;
      }
      int64_t v = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        long long n2 = __shfl_up_sync(0xffffffffu, (long long)v, o);
        if (lane >= o) v += n2;
      }
      if (lane == 31) wsum[warp] = v;
      __syncthreads();
      int64_t off = 0;
      for (int w = 0; w < warp; w++) off += wsum[w];
      if (tid < nmem) pref[tid + 1] = v + off;
      if (tid == 0) pref[0] = 0;
      __syncthreads();
      const int64_t total = pref[nmem];
      for (int64_t p0 = 0; p0 < total; p0 += TILE) {
        const int cnt = (int)(total - p0 < TILE ? total - p0 : TILE);
        for (int t = tid; t < cnt; t += IT2) {
          const int64_t p = p0 + t;
          int lo = 0, hi = nmem;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (pref[mid] <= p) lo = mid;
            else hi = mid;
          }
          const int64_t src = sbeg[lo] + (p - pref[lo]);
          double rec[2 * W];
#pragma unroll
          for (int k = 0; k < D; k++) rec[k] = __ldg(T.sc + k * T.ld_s + src);
#pragma unroll
          for (int r = 0; r < NR; r++) rec[D + r] = __ldg(T.q + src * R + r0 + r);
#pragma unroll
          for (int k = D + NR; k < 2 * W; k++) rec[k] = 0.0;
#pragma unroll
          for (int w = 0; w < W; w++) tile[t * W + w] = make_double2(rec[2 * w], rec[2 * w + 1]);
        }
        __syncthreads();
        if (worker) {
          for (int j = grp; j < cnt; j += G) {
            double rec[2 * W];
#pragma unroll
            for (int w = 0; w < W; w++) {
              const double2 u2 = tile[j * W + w];
              rec[2 * w] = u2.x;
              rec[2 * w + 1] = u2.y;
            }
#pragma unroll
            for (int t = 0; t < RT; t++) {
              double r2 = 0.0;
#pragma unroll
              for (int k = 0; k < D; k++) {
                const double dk = x[t][k] - rec[k];
                r2 = fma(dk, dk, r2);
              }
              double kv;
              if constexpr ((KIND == COULOMB || KIND == LAPLACE) && !SELF) {
                const double y = rsq_approx(r2);
                const double e = fma(-r2, y * y, 1.0);
                kv = fma(y * e, fma(0.375, e, 0.5), y);
              } else {
                kv = kpair<KIND>(r2, kp);
              }
#pragma unroll
              for (int r = 0; r < NR; r++) acc[t][r] = fma(kv, rec[D + r], acc[t][r]);
            }
          }
        }
        __syncthreads();
      }
    }
#pragma unroll
    for (int t = 0; t < RT; t++)
#pragma unroll
      for (int r = 0; r < NR; r++) part[(t * IT2 + tid) * NR + r] = acc[t][r];
    __syncthreads();
    if (worker && grp == 0) {
#pragma unroll
      for (int t = 0; t < RT; t++) {
        if (!act[t]) continue;
        const int64_t a = a0 + slot + t * TS;
#pragma unroll
        for (int r = 0; r < NR; r++) {
          double tot = 0.0;
          for (int g = 0; g < G; g++) tot += part[(t * IT2 + g * TS + slot) * NR + r];
          T.out[(tb + a) * R + r0 + r] = tot * kscale<KIND>();
        }
      }
    }
    __syncthreads();
  }
}

template <int D, int KIND, int NR, int TILE, int RT>
__global__ void __launch_bounds__(IT2) interact2(const int64_t* __restrict__ items,
                                                 const LevelTab* __restrict__ tabs, int near_list, int64_t R,
                                                 int64_t r0, KParams kp) {
  constexpr int W = SrcW<D, NR>::W;
  __shared__ double2 tile[W * TILE];
  __shared__ int64_t pref[MAXMEM + 1];
  __shared__ int64_t sbeg[MAXMEM];
  __shared__ int64_t wsum[IT2 / 32];
  __shared__ double part[2 * IT2 * NR];
  const int64_t it = items[blockIdx.x];
  const int lev = (int)(it >> 40);
  const int64_t c = it & ((1ll << 40) - 1);
  const LevelTab T = tabs[lev];
  if (lev == near_list)
    interact_cell<D, KIND, NR, TILE, true, RT>(T, c, R, r0, kp, tile, pref, sbeg, wsum, part);
  else
    interact_cell<D, KIND, NR, TILE, false, RT>(T, c, R, r0, kp, tile, pref, sbeg, wsum, part);
}

template <int D, int KIND, int NR, int TILE>
void launch_chunk(const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  if (!h.n_items) return;
  const unsigned g = (unsigned)h.n_items;
  const int nl = h.t->depth + 1;  // list id of the leaf near field
  auto* items = h.items.get();
  auto* tabs = reinterpret_cast<const LevelTab*>(h.tabs.get());
  interact2<D, KIND, NR, TILE, 2><<<g, IT2, 0, s>>>(items, tabs, nl, R, r0, kp);
  CKL();
}

template <int D, int KIND>
void launch_interact2(const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp, cudaStream_t s) {
  if (nr == 16) launch_chunk<D, KIND, 16, 64>(h, R, r0, kp, s);
  else launch_chunk<D, KIND, 1, H2B_TILE1>(h, R, r0, kp, s);
}

template <int D>
void interact_all_d_impl(int kind, const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp,
                         cudaStream_t s) {
  switch (kind) {
    case COULOMB: launch_interact2<D, COULOMB>(h, R, r0, nr, kp, s); break;
    case LAPLACE: launch_interact2<D, LAPLACE>(h, R, r0, nr, kp, s); break;
    case GAUSSIAN: launch_interact2<D, GAUSSIAN>(h, R, r0, nr, kp, s); break;
    case GAUSSIAN_SCALED: launch_interact2<D, GAUSSIAN_SCALED>(h, R, r0, nr, kp, s); break;
    case MATERN: launch_interact2<D, MATERN>(h, R, r0, nr, kp, s); break;
    case LOG: launch_interact2<D, LOG>(h, R, r0, nr, kp, s); break;
    case REG_INVERSE: launch_interact2<D, REG_INVERSE>(h, R, r0, nr, kp, s); break;
    default: launch_interact2<D, REG_LOG>(h, R, r0, nr, kp, s); break;
  }
}

}  // namespace

template <int D>
void interact_all_d(int kind, const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp, cudaStream_t s);

}  // namespace h2b
