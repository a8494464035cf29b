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


namespace {

// ---------------------------------------------------------------------
// Interaction kernel: one launch for every M2L level and the near field.
//
// Work item = (list, cell): list l in [2, L] is level l's interaction list
// (targets = the cell's incoming pivots, sources = outgoing pivots of the
// interaction-list cells, charges = their multipole coefficients); list
// L + 1 is the leaf near field (points and input charges).  Items are sorted
// by pair count, largest first, so all levels share one balanced grid.
//
// A CTA owns one target cell.  Its targets sit in registers (2 per thread);
// the sources are packed records [x, y, z, q...] streamed into shared memory
// with cp.async (double-buffered tiles) and read back as LDS.128 broadcasts.
// ---------------------------------------------------------------------
#ifndef H2B_IT2
#define H2B_IT2 128
#endif
#ifndef H2B_TILE1
#define H2B_TILE1 256
#endif
constexpr int IT2 = H2B_IT2;
constexpr int MEMPT = 2;                 // list members per thread in the prefix scan
constexpr int MAXMEM = IT2 * MEMPT;      // list members per chunk

struct LevelTab {
  const double* tc;      // target coords SoA (ld_t)
  int64_t ld_t;
  const int64_t* t_ptr;  // target range per cell
  int64_t rec_off;       // first source record of this list
  const int64_t* s_ptr;  // source range per source cell
  const int64_t* l_ptr;  // cell list (CSR)
  const int64_t* l_idx;
  double* out;           // result rows (target position) * R
};

struct PackTab {
  const double* sc;  // source coords SoA
  int64_t ld_s;
  const double* q;   // charges (row stride R)
  int64_t n;         // sources in this list
  int64_t rec_off;
};

__device__ __forceinline__ double rsq_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// 1/r without the diagonal test: MUFU.RSQ64H seed + cubic Newton correction
__device__ __forceinline__ double rsqrt_full(double r2) {
  const double y = rsq_approx(r2);
  const double e = fma(-r2, y * y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}

// K(r2) with the punctured diagonal (near field may pair a point with itself)
template <int KIND>
__device__ __forceinline__ double kpair(double r2, const KParams& kp) {
  if constexpr (KIND == COULOMB || KIND == LAPLACE) {
    const bool zero = __double2hiint(r2) == 0;  // r2 == 0 (or subnormal)
    const double kv = rsqrt_full(zero ? 1.0 : r2);
    return zero ? 0.0 : kv;
  } else {
    return kfast<KIND>(r2, kp);
  }
}

// record = [y_0..y_{D-1}, q_0..q_{NR-1}, |y|^2], padded to whole double2 words
template <int D, int NR>
struct SrcW {
  static constexpr int W = (D + NR + 2) / 2;  // double2 words per source record
};

template <int D, int NR>
__global__ void pack_records(const PackTab* __restrict__ pt, int nlists, int64_t total, int64_t R, int64_t r0,
                             double2* __restrict__ rec) {
  constexpr int W = SrcW<D, NR>::W;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= total) return;
  int l = 0;
  while (l + 1 < nlists && pt[l + 1].rec_off <= p) l++;
  const PackTab T = pt[l];
  const int64_t i = p - T.rec_off;
  double v[2 * W];
  double n2 = 0.0;
#pragma unroll
  for (int k = 0; k < D; k++) {
    v[k] = T.sc[k * T.ld_s + i];
    n2 = fma(v[k], v[k], n2);
  }
#pragma unroll
  for (int r = 0; r < NR; r++) v[D + r] = T.q[i * R + r0 + r];
  v[D + NR] = n2;
#pragma unroll
  for (int k = D + NR + 1; k < 2 * W; k++) v[k] = 0.0;
#pragma unroll
  for (int w = 0; w < W; w++) rec[p * W + w] = make_double2(v[2 * w], v[2 * w + 1]);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Copy source records [p0, p0 + cnt) of the flattened list into a tile:
// warps take the list members that intersect the window round-robin and
// their lanes issue one 16-byte cp.async per record word.
template <int W, int TILE>
__device__ __forceinline__ void fill_tile(double2* dst, const double2* __restrict__ rec, int64_t p0, int cnt,
                                          const int64_t* pref, const int64_t* sbeg, int nmem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int lo = 0, hi = nmem;  // first member with pref[q + 1] > p0  <=>  last q with pref[q] <= p0
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (pref[mid] <= p0) lo = mid;
    else hi = mid;
  }
  const int64_t p1 = p0 + cnt;
  for (int q = lo + warp; q < nmem && pref[q] < p1; q += IT2 / 32) {
    const int64_t a = pref[q] > p0 ? pref[q] : p0;
    const int64_t b = pref[q + 1] < p1 ? pref[q + 1] : p1;
    const double2* src = rec + (sbeg[q] + (a - pref[q])) * W;
    double2* d = dst + (a - p0) * W;
    const int nw = (int)(b - a) * W;
    for (int e = lane; e < nw; e += 32) cp_async16(d + e, src + e);
  }
  cp_async_commit();
}

// One pair.  Near field (SELF): r^2 from coordinate differences.  Interaction
// lists (separated cells, r >= one cell width): r^2 = |x|^2 + |y|^2 - 2 x.y
// with xm2 = -2x precomputed, 4 FP64 ops instead of 6; the cancellation error
// is <= 1e-16 (|x|^2 + |y|^2) / r^2 ~ 1e-12 relative at the finest level.
template <int D, int KIND, int NR, bool SELF>
__device__ __forceinline__ void pair_accum(const double (&x)[D], const double (&xm2)[D], double nx,
                                           const double* rec, double (&acc)[NR], const KParams& kp) {
  double r2;
  if constexpr (SELF) {
    r2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; k++) {
      const double dk = x[k] - rec[k];
      r2 = fma(dk, dk, r2);
    }
  } else {
    r2 = nx + rec[D + NR];
#pragma unroll
    for (int k = 0; k < D; k++) r2 = fma(xm2[k], rec[k], r2);
  }
  double kv;
  if constexpr ((KIND == COULOMB || KIND == LAPLACE) && !SELF) kv = rsqrt_full(r2);
  else kv = kpair<KIND>(r2, kp);
#pragma unroll
  for (int r = 0; r < NR; r++) acc[r] = fma(kv, rec[D + r], acc[r]);
}

// SELF = the list may contain the target itself (near field).
template <int D, int KIND, int NR, int TILE, bool SELF, int RT>
__device__ __forceinline__ void interact_cell(const LevelTab& T, const double2* __restrict__ rec, int64_t c,
                                              int64_t R, int64_t r0, const KParams& kp, double2* tiles,
                                              int64_t* pref, int64_t* sbeg, int64_t* wsum, double* part) {
  constexpr int W = SrcW<D, NR>::W;
  const int64_t tb = T.t_ptr[c], m = T.t_ptr[c + 1] - tb;
  const int64_t lb = T.l_ptr[c], le = T.l_ptr[c + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double2* lrec = rec + T.rec_off * W;
  for (int64_t a0 = 0; a0 < m; a0 += RT * IT2) {
    const int64_t mc = (m - a0) < RT * IT2 ? (m - a0) : RT * IT2;
    const int TS = (int)((mc + RT - 1) / RT);
    const int G = IT2 / TS;
    const int slot = tid % TS, grp = tid / TS;
    const bool worker = grp < G;
    bool act[RT];
    double x[RT][D], xm2[RT][D], nx[RT];
    double acc[RT][NR];
#pragma unroll
    for (int t = 0; t < RT; t++) {
      const int64_t a = a0 + slot + t * TS;
      act[t] = worker && (slot + t * TS) < mc;
      nx[t] = 0.0;
#pragma unroll
      for (int k = 0; k < D; k++) {
        x[t][k] = act[t] ? T.tc[k * T.ld_t + tb + a] : 0.0;
        xm2[t][k] = -2.0 * x[t][k];
        nx[t] = fma(x[t][k], x[t][k], nx[t]);
      }
#pragma unroll
      for (int r = 0; r < NR; r++) acc[t][r] = 0.0;
    }
    for (int64_t q0 = lb; q0 < le; q0 += MAXMEM) {
      const int nmem = (int)(le - q0 < MAXMEM ? le - q0 : MAXMEM);
      // exclusive prefix of member lengths: MEMPT members per thread + block scan
      int64_t loc[MEMPT];
      int64_t run = 0;
#pragma unroll
      for (int u = 0; u < MEMPT; u++) {
        const int q = tid * MEMPT + u;
        int64_t len = 0;
        if (q < nmem) {
          const int64_t sc = T.l_idx[q0 + q];
          const int64_t b = T.s_ptr[sc];
          sbeg[q] = b;
          len = T.s_ptr[sc + 1] - b;
        }
        loc[u] = run;
        run += len;
      }
      int64_t v = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long n2 = __shfl_up_sync(0xffffffffu, (long long)v, o);
        if (lane >= o) v += n2;
      }
      if (lane == 31) wsum[warp] = v;
      __syncthreads();
      int64_t off = v - run;
      for (int w = 0; w < warp; w++) off += wsum[w];
#pragma unroll
      for (int u = 0; u < MEMPT; u++) {
        const int q = tid * MEMPT + u;
        if (q <= nmem) pref[q] = off + loc[u];
      }
      if (tid == IT2 - 1 && nmem == MAXMEM) pref[MAXMEM] = off + run;
      __syncthreads();
      const int64_t total = pref[nmem];
      const int ntile = (int)((total + TILE - 1) / TILE);
      if (ntile > 0) fill_tile<W, TILE>(tiles, lrec, 0, (int)(total < TILE ? total : TILE), pref, sbeg, nmem);
      for (int it = 0; it < ntile; it++) {
        const int64_t p0 = (int64_t)it * TILE;
        const int cnt = (int)(total - p0 < TILE ? total - p0 : TILE);
        double2* cur = tiles + (it & 1) * TILE * W;
        if (it + 1 < ntile) {
          const int64_t p1 = p0 + TILE;
          fill_tile<W, TILE>(tiles + ((it + 1) & 1) * TILE * W, lrec, p1,
                             (int)(total - p1 < TILE ? total - p1 : TILE), pref, sbeg, nmem);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        if (worker) {
          int j = grp;
          for (; j + G < cnt; j += 2 * G) {
            double ra[2 * W], rb[2 * W];
#pragma unroll
            for (int w = 0; w < W; w++) {
              const double2 ua = cur[j * W + w], ub = cur[(j + G) * W + w];
              ra[2 * w] = ua.x;
              ra[2 * w + 1] = ua.y;
              rb[2 * w] = ub.x;
              rb[2 * w + 1] = ub.y;
            }
#pragma unroll
            for (int t = 0; t < RT; t++) {
              pair_accum<D, KIND, NR, SELF>(x[t], xm2[t], nx[t], ra, acc[t], kp);
              pair_accum<D, KIND, NR, SELF>(x[t], xm2[t], nx[t], rb, acc[t], kp);
            }
          }
          if (j < cnt) {
            double ra[2 * W];
#pragma unroll
            for (int w = 0; w < W; w++) {
              const double2 ua = cur[j * W + w];
              ra[2 * w] = ua.x;
              ra[2 * w + 1] = ua.y;
            }
#pragma unroll
            for (int t = 0; t < RT; t++) pair_accum<D, KIND, NR, SELF>(x[t], xm2[t], nx[t], ra, acc[t], kp);
          }
        }
        __syncthreads();
      }
    }
#pragma unroll
    for (int t = 0; t < RT; t++) {
#pragma unroll
      for (int r = 0; r < NR; r++) part[tid * NR + r] = acc[t][r];
      __syncthreads();
      if (worker && grp == 0 && act[t]) {
        const int64_t a = a0 + slot + t * TS;
#pragma unroll
        for (int r = 0; r < NR; r++) {
          double tot = 0.0;
          for (int g = 0; g < G; g++) tot += part[(g * TS + slot) * NR + r];
          T.out[(tb + a) * R + r0 + r] = tot * kscale<KIND>();
        }
      }
      __syncthreads();
    }
  }
}

template <int D, int KIND, int NR, int TILE, int RT>
__global__ void __launch_bounds__(IT2) interact2(const int64_t* __restrict__ items,
                                                 const LevelTab* __restrict__ tabs, const double2* __restrict__ rec,
                                                 int near_list, int64_t R, int64_t r0, KParams kp) {
  constexpr int W = SrcW<D, NR>::W;
  __shared__ __align__(16) double2 tiles[2 * W * TILE];
  __shared__ int64_t pref[MAXMEM + 1];
  __shared__ int64_t sbeg[MAXMEM];
  __shared__ int64_t wsum[IT2 / 32];
  __shared__ double part[IT2 * NR];
  const int64_t it = items[blockIdx.x];
  const int lev = (int)(it >> 40);
  const int64_t c = it & ((1ll << 40) - 1);
  const LevelTab T = tabs[lev];
  if (lev == near_list)
    interact_cell<D, KIND, NR, TILE, true, RT>(T, rec, c, R, r0, kp, tiles, pref, sbeg, wsum, part);
  else
    interact_cell<D, KIND, NR, TILE, false, RT>(T, rec, c, R, r0, kp, tiles, pref, sbeg, wsum, part);
}

template <int D, int KIND, int NR, int TILE>
void launch_chunk(const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  constexpr int W = SrcW<D, NR>::W;
  const int L = h.t->depth;
  double2* rec = reinterpret_cast<double2*>(h.rec.get());
  pack_records<D, NR><<<ceil_div(h.rec_total, 256), 256, 0, s>>>(
      reinterpret_cast<const PackTab*>(h.packtab.get()), L + 2, h.rec_total, R, r0, rec);
  CKL();
  if (!h.n_items) return;
  (void)W;
  const unsigned g = (unsigned)h.n_items;
  auto* items = h.items.get();
  auto* tabs = reinterpret_cast<const LevelTab*>(h.tabs.get());
  if constexpr (NR == 1) {
    static const int rt = [] {
      const char* e = getenv("H2B_RT");
      return e ? atoi(e) : 2;
    }();
    if (rt == 1) interact2<D, KIND, NR, TILE, 1><<<g, IT2, 0, s>>>(items, tabs, rec, L + 1, R, r0, kp);
    else if (rt == 4) interact2<D, KIND, NR, TILE, 4><<<g, IT2, 0, s>>>(items, tabs, rec, L + 1, R, r0, kp);
    else interact2<D, KIND, NR, TILE, 2><<<g, IT2, 0, s>>>(items, tabs, rec, L + 1, R, r0, kp);
  } else {
    interact2<D, KIND, NR, TILE, 2><<<g, IT2, 0, s>>>(items, tabs, rec, L + 1, R, r0, kp);
  }
  CKL();
}

template <int D, int KIND>
void launch_interact2(const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp, cudaStream_t s) {
  if (nr == 16) launch_chunk<D, KIND, 16, 32>(h, R, r0, kp, s);
  else launch_chunk<D, KIND, 1, H2B_TILE1>(h, R, r0, kp, s);
}

template <int D>
void interact_all_d_impl(int kind, const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp, cudaStream_t s) {
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
