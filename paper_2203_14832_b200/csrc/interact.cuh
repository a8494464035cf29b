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

// exp(x) for the Gaussian / Matern kernels' x = -a r^2, -r <= 0 (matvec path).  Table
// reduction x = (16 m + j) ln2/16 + r, |r| <= ln2/32: exp(x) = 2^m 2^(j/16)
// exp(r), exp(r) by its degree-7 Taylor polynomial (truncation r^8/8! <=
// 5e-19), 2^(j/16) from a 16-entry table of correctly rounded doubles (one
// 128-byte L1 line: every lane pattern is one request), 2^m folded into the
// table entry's exponent.  12 FP64 instructions and no slow-path branches
// instead of the ~25 of CUDA's exp; error ~2 ulp.  x < -708 (exp < 3.3e-308)
// returns 0.
__device__ __align__(128) const double kExp2Tab16[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};

__device__ __forceinline__ double exp_neg_fast(double x) {
  constexpr double MAGIC = 0x1.8p52;             // round-to-integer shifter
  constexpr double INV = 23.083120654223414;     // 16 / ln 2
  constexpr double C_HI = 0.04332169878499658;   // ln2 / 16, head
  constexpr double C_LO = 1.4494042586539372e-18;  // ln2 / 16, tail
  const double t = fma(x, INV, MAGIC);
  const int n = __double2loint(t);  // round(x * 16 / ln2)
  const double nd = t - MAGIC;
  double r = fma(nd, -C_HI, x);
  r = fma(nd, -C_LO, r);
  double p = fma(r, 1.0 / 5040.0, 1.0 / 720.0);
  p = fma(r, p, 1.0 / 120.0);
  p = fma(r, p, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = fma(r, p, 1.0);
  const double tj = __ldg(&kExp2Tab16[n & 15]);
  const double sj = __hiloint2double(__double2hiint(tj) + (n >> 4) * (1 << 20), __double2loint(tj));
  return x < -708.0 ? 0.0 : sj * p;
}

// fast kernel evaluation (matvec path; tolerance 1e-10 relative)
template <int KIND>
__device__ __forceinline__ double kfast(double r2, const KParams& kp) {
  if constexpr (KIND == COULOMB || KIND == LAPLACE) {
    return r2 > 0.0 ? rsqrt(r2) : 0.0;  // LAPLACE's 1/(4 pi) applied to the sum
  } else if constexpr (KIND == GAUSSIAN) {
    return exp_neg_fast(-r2);
  } else if constexpr (KIND == GAUSSIAN_SCALED) {
    return exp_neg_fast(-kp.a * r2);
  } else if constexpr (KIND == MATERN) {
    return exp_neg_fast(-sqrt(r2));
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
// target cell: RT targets per thread in registers; the sources are streamed
// through shared memory as packed records [y_0..y_{D-1}, q_0..q_{NR-1}]
// (source records, `SrcRec`): every list member's sources are one contiguous
// record range (Morton cell order), so a tile is filled by one TMA bulk copy
// (cp.async.bulk, mbarrier completion) per member, double-buffered so the
// copy of tile i+1 overlaps the arithmetic of tile i.
// ---------------------------------------------------------------------
namespace {

#ifndef H2B_IT2
#define H2B_IT2 128
#endif
#ifndef H2B_RT
#define H2B_RT 3  // largest targets per lane (one-RHS kernel); 2 for multi-RHS
#endif
#ifndef H2B_UNROLL
#define H2B_UNROLL 2
#endif
#ifndef H2B_MINB
#define H2B_MINB 4  // 4 CTAs x 4 warps per SM (caps registers at 128)
#endif
#ifndef H2B_TILE16
#define H2B_TILE16 32
#endif
#ifndef H2B_TILE1
#define H2B_TILE1 128
#endif
constexpr int IT2 = H2B_IT2;
#ifndef H2B_MAXMEMW
#define H2B_MAXMEMW 256
#endif
constexpr int MAXMEMW = H2B_MAXMEMW;
constexpr int UNROLL_J = H2B_UNROLL;  // source-loop unroll (independent pair chains per lane)

// doubles per source record (padded to whole 16-byte words for TMA / LDS.128)
template <int D, int NR>
struct SrcRec {
  static constexpr int RS = 2 * ((D + NR + 1) / 2);
  static constexpr int W = RS / 2;  // double2 words
};

struct LevelTab {
  const double* tc;      // target coords SoA (ld_t)
  int64_t ld_t;
  const int64_t* t_ptr;  // target range per cell
  const int64_t* s_ptr;  // source range per source cell (record index)
  const double2* rec1;   // source records for NR = 1
  const double2* rec16;  // source records for NR = 16
  const int64_t* l_ptr;  // cell list (CSR)
  const int64_t* l_idx;
  const int* m_sb;       // per list entry: first record of the member
  const int* m_end;      // per member: inclusive prefix of member lengths within the cell's list
  const int* m_cnt;      // members per cell (compacted at the head of the cell's list segment; adjacent
                         // record ranges merged; near field: the cell itself is dropped, it has its own pass)
  double* out;           // result rows (target position) * R
};

__device__ __forceinline__ double rsq_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// M2L seed from the FP32 MUFU: the double's exponent is rebased to FP32
// (1023 -> 127) and its mantissa truncated to 23 bits in integer arithmetic
// (funnel shift + add, no F2F conversion), rsqrt.approx.f32 (max rel error
// 2^-22.9), then widened back the same way.  Seed error |d| <= 1.8e-7 (vs
// 9.2e-7 for MUFU.RSQ64H), so one quadratic Newton step (relative error
// 1.5 d^2 <= 5e-14) replaces the cubic one: 2 fewer FP64 instructions per
// pair.  Valid for r2 in [2^-126, 2^127]: the host selects this path only
// when the tree's geometry bounds every admissible pair inside
// [2^-100, 2^100] (f32seed_ok in launch_chunk).
__device__ __forceinline__ double rsq_seed_f32(double x) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const int fb = (int)__funnelshift_l((unsigned)lo, (unsigned)hi, 3) - ((1023 - 127) << 23);
  float yf;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(yf) : "f"(__int_as_float(fb)));
  const int yb = __float_as_int(yf);
  return __hiloint2double((int)((unsigned)yb >> 3) + ((1023 - 127) << 20), yb << 29);
}

// K(r2) for the interaction kernel, non-1/r kinds (1/r is acc_inv_r).
template <int KIND>
__device__ __forceinline__ double kpair(double r2, const KParams& kp) {
  return kfast<KIND>(r2, kp);
}

// r^2 of one pair.
//   SELF (near field): coordinate differences, so identical points give
//   exactly 0 (the punctured diagonal).
//   Interaction lists (admissible, separated cells): both sides are shifted to
//   the origin o = the first target of the CTA's cell, and
//   r^2 = |x'|^2 + |y'|^2 - 2 x'.y'  costs 4 FP64 ops (DADD + 3 DFMA) instead
//   of 6.  The cancellation error is ~eps (|x'|^2 + |y'|^2) / r^2 ~ 1e-15
//   relative: |x'| <= diam(X), |y'| <= dist + 2 diam, and admissibility
//   bounds diam / dist (measured: matvec error vs the oracle unchanged).
template <int D, bool SELF>
__device__ __forceinline__ double pair_r2(const double (&x)[D + 1], const double* rec, double yy) {
  if constexpr (SELF) {
    double r2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; k++) {
      const double dk = x[k] - rec[k];
      r2 = fma(dk, dk, r2);
    }
    return r2;
  } else {
    double r2 = x[D] + yy;  // |x'|^2 + |y'|^2
#pragma unroll
    for (int k = 0; k < D; k++) r2 = fma(x[k], rec[k], r2);  // x holds -2 x'
    return r2;
  }
}

// Accumulate q K(r2) for 1/r (COULOMB / LAPLACE) in "2/r" units (the sum is
// scaled by 1/2 at the end), from the MUFU.RSQ64H seed y (relative error
// <= 9.2e-7, tools/ubench_rsq.cu).
//   M2L (!SELF): cubic correction  2/r = y (2 + e + 3/4 e^2), e = 1 - r2 y^2
//   (<= 1 ulp).  The multipole charges come from interpolation weights with
//   cancellation, so a one-sided per-entry bias is amplified: a quadratic
//   step (error 1.5 e^2 <= 1.3e-12 per entry) measured 2.5e-11 against the
//   oracle at N = 1M, the cubic one 1.5e-13.
//   Near field (SELF, plain input charges): quadratic step 2/r = y (3 - r2 y^2).
//   TEST: the source range may hold the target itself or a duplicate point,
//   r2 == 0 -> K = 0 (the punctured diagonal); only the target's own leaf can,
//   so only that member pays for the test.
template <int NR, bool SELF, bool TEST, bool F32S>
__device__ __forceinline__ void acc_inv_r(double r2, const double* q, double (&acc)[NR]) {
  if constexpr (TEST) {
    const bool zero = __double2hiint(r2) == 0;  // r2 == 0 (or subnormal)
    const double r2s = zero ? 1.0 : r2;
    const double y = rsq_approx(r2s);
    const double t = fma(-r2s, y * y, 3.0);
    const double kv = zero ? 0.0 : y * t;
#pragma unroll
    for (int r = 0; r < NR; r++) acc[r] = fma(kv, q[r], acc[r]);
  } else {
    const double y = (F32S && !SELF) ? rsq_seed_f32(r2) : rsq_approx(r2);
    double t;
    if constexpr (SELF || F32S) {
      t = fma(-r2, y * y, 3.0);
    } else {
      const double e = fma(-r2, y * y, 1.0);
      t = fma(e, fma(0.75, e, 1.0), 2.0);
    }
    if constexpr (NR == 1) {
      acc[0] = fma(y * q[0], t, acc[0]);
    } else {
      const double kv = y * t;
#pragma unroll
      for (int r = 0; r < NR; r++) acc[r] = fma(kv, q[r], acc[r]);
    }
  }
}

template <int KIND>
__device__ __forceinline__ constexpr bool is_inv_r() {
  return KIND == COULOMB || KIND == LAPLACE;
}

// Per-warp shared-memory state.  Every warp is an independent worker (no
// CTA-wide barriers in the source loop): it owns two TMA stages, their
// mbarriers and its list-member table.
template <int D, int NR, int TILE, int RT>
struct WarpSmem {
  static constexpr int W = SrcRec<D, NR>::W;
  static constexpr int RTMAX = RT;
  double2 stage[2][TILE * W];  // TMA destinations (double-buffered)
  double yy[TILE];             // |y'|^2 of the current tile (interaction lists)
  uint64_t bar[2];             // "tile landed" mbarriers
  int pref[MAXMEMW + 1];       // prefix of member lengths (records)
  int sbeg[MAXMEMW];           // first record of each member (records < 2^31, checked on the host)
  double part[RT * 32 * NR];   // per-group partial sums
};

// Issue the TMA bulk copies of window [p0, p0 + cnt) of the member
// concatenation into one stage (whole warp; lane 0 arms the mbarrier first).
template <int W>
__device__ __forceinline__ void issue_tile(const double2* rec, int nmem, const int* pref, const int* sbeg,
                                           int p0, int cnt, double2* dst, uint64_t* bar, int& lo) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) mbar_expect_tx(bar, (uint32_t)cnt * (uint32_t)(W * 16));
  __syncwarp();
  // windows advance monotonically: lo (warp-uniform) = a member at or before the one holding p0
  while (pref[lo + 1] <= p0) lo++;
  const int p1 = p0 + cnt;
  int last = lo;
  for (int qm = lo + lane; qm < nmem && pref[qm] < p1; qm += 32) {
    const int pa = pref[qm] > p0 ? pref[qm] : p0;
    const int pb = pref[qm + 1] < p1 ? pref[qm + 1] : p1;
    last = qm;
    if (pb > pa)
      bulk_g2s(dst + (pa - p0) * W, rec + (int64_t)(sbeg[qm] + (pa - pref[qm])) * W, (uint32_t)(pb - pa) * (W * 16), bar);
  }
  lo = __reduce_max_sync(0xffffffffu, last);  // the member holding the end of this window
}

// Stream the concatenated source ranges of nmem list members (sbeg / pref in
// the warp's shared memory) through the double-buffered tiles and accumulate
// into the register-resident targets.  `ntile` counts the tiles this warp
// has consumed (stage = ntile & 1, mbarrier parity = (ntile >> 1) & 1).
template <int D, int KIND, int NR, int TILE, bool SELF, bool TEST, int RT, bool F32S, class WS>
__device__ __forceinline__ void stream_members(WS& S, const double2* rec, int nmem,
                                               const double (&o)[D], const KParams& kp, bool worker, int grp,
                                               int G, const double (&x)[RT][D + 1], double (&acc)[RT][NR],
                                               uint32_t& ntile) {
  constexpr int W = SrcRec<D, NR>::W;
  const int lane = threadIdx.x & 31;
  const int total = S.pref[nmem];
  if (total == 0) return;
  const int ntiles = (total + TILE - 1) / TILE;
  int lo = 0;  // issue cursor over the members
  issue_tile<W>(rec, nmem, S.pref, S.sbeg, 0, total < TILE ? total : TILE, S.stage[ntile & 1], &S.bar[ntile & 1], lo);
  for (int it = 0; it < ntiles; it++, ntile++) {
    const int b = ntile & 1;
    const int p0 = it * TILE;
    const int cnt = total - p0 < TILE ? total - p0 : TILE;
    double2* tile = S.stage[b];
    mbar_wait(&S.bar[b], (ntile >> 1) & 1);
    if constexpr (!SELF) {  // shift to the target-cell origin in place, |y'|^2 aside
      for (int e = lane; e < cnt; e += 32) {
        double v[2 * W];
#pragma unroll
        for (int w = 0; w < W; w++) {
          const double2 u2 = tile[e * W + w];
          v[2 * w] = u2.x;
          v[2 * w + 1] = u2.y;
        }
        double n2 = 0.0;
#pragma unroll
        for (int k = 0; k < D; k++) {
          v[k] -= o[k];
          n2 = fma(v[k], v[k], n2);
        }
        S.yy[e] = n2;
#pragma unroll
        for (int w = 0; w < (D + 1) / 2; w++) tile[e * W + w] = make_double2(v[2 * w], v[2 * w + 1]);
      }
      fence_proxy_async();
      __syncwarp();
    }
    // next tile into the other stage (its last reader finished before the __syncwarp closing the previous tile)
    if (it + 1 < ntiles) {
      const int q0 = p0 + TILE;
      issue_tile<W>(rec, nmem, S.pref, S.sbeg, q0, total - q0 < TILE ? total - q0 : TILE, S.stage[b ^ 1],
                    &S.bar[b ^ 1], lo);
    }
    if (worker) {
#pragma unroll (UNROLL_J)
      for (int j = grp; j < cnt; j += G) {
        double v[2 * W];
#pragma unroll
        for (int w = 0; w < W; w++) {
          const double2 u2 = tile[j * W + w];
          v[2 * w] = u2.x;
          v[2 * w + 1] = u2.y;
        }
        const double yy = SELF ? 0.0 : S.yy[j];
#pragma unroll
        for (int t = 0; t < RT; t++) {
          const double r2 = pair_r2<D, SELF>(x[t], v, yy);
          if constexpr (is_inv_r<KIND>()) {
            acc_inv_r<NR, SELF, TEST, F32S>(r2, v + D, acc[t]);
          } else {
            const double kv = kpair<KIND>(r2, kp);
#pragma unroll
            for (int r = 0; r < NR; r++) acc[t][r] = fma(kv, v[D + r], acc[t][r]);
          }
        }
      }
    }
    __syncwarp();
  }
}

// One work item (list, cell) on one warp.  RT targets per lane (register
// blocking: every shared-memory source read feeds RT pair evaluations), TS
// lanes per target group, G = 32 / TS groups splitting the sources.  Near
// field (SELF): the target's own leaf goes first through the r2 == 0 test
// path, the other neighbours (never coincident with a target) through the
// plain path.
template <int D, int KIND, int NR, int TILE, bool SELF, int RT, bool F32S, class WS>
__device__ __forceinline__ void interact_cell_rt(const LevelTab& T, int64_t c, const int4 dsc, int64_t R, int64_t r0,
                                                 const KParams& kp, WS& S, uint32_t& ntile) {
  const double2* rec = NR == 1 ? T.rec1 : T.rec16;
  const int64_t tb = dsc.x, m = dsc.y, lb = dsc.z, le = dsc.w;  // precomputed item descriptor
  const int lane = threadIdx.x & 31;
  double o[D];
#pragma unroll
  for (int k = 0; k < D; k++) o[k] = SELF ? 0.0 : T.tc[k * T.ld_t + tb];
  for (int64_t a0 = 0; a0 < m; a0 += RT * 32) {
    const int64_t mc = (m - a0) < RT * 32 ? (m - a0) : RT * 32;
    const int TS = (int)((mc + RT - 1) / RT);
    const int G = 32 / TS;
    const int slot = lane % TS, grp = lane / TS;
    const bool worker = grp < G;
    bool act[RT];
    double x[RT][D + 1];
    double acc[RT][NR];
#pragma unroll
    for (int t = 0; t < RT; t++) {
      const int64_t a = a0 + slot + t * TS;
      act[t] = worker && (slot + t * TS) < mc;
      double n2 = 0.0;
#pragma unroll
      for (int k = 0; k < D; k++) {
        const double xk = act[t] ? T.tc[k * T.ld_t + tb + a] : o[k];
        if constexpr (SELF) {
          x[t][k] = xk;
        } else {
          const double dk = xk - o[k];
          n2 = fma(dk, dk, n2);
          x[t][k] = -2.0 * dk;
        }
      }
      x[t][D] = n2;
#pragma unroll
      for (int r = 0; r < NR; r++) acc[t][r] = 0.0;
    }
    if constexpr (SELF) {  // own leaf: the only member that can hold r2 == 0
      if (lane == 0) {
        const int64_t b = T.s_ptr[c];
        S.sbeg[0] = (int)b;
        S.pref[0] = 0;
        S.pref[1] = (int)(T.s_ptr[c + 1] - b);
      }
      __syncwarp();
      stream_members<D, KIND, NR, TILE, SELF, true, RT, F32S>(S, rec, 1, o, kp, worker, grp, G, x, acc, ntile);
    }
    for (int64_t q0 = lb; q0 < le; q0 += MAXMEMW) {
      const int nmem = (int)(le - q0 < MAXMEMW ? le - q0 : MAXMEMW);
      {  // member table of this chunk from the precomputed per-entry arrays (one coalesced round trip)
        const int base = q0 == lb ? 0 : T.m_end[q0 - 1];
        for (int i = lane; i < nmem; i += 32) {
          S.sbeg[i] = T.m_sb[q0 + i];
          S.pref[i + 1] = T.m_end[q0 + i] - base;
        }
        if (lane == 0) S.pref[0] = 0;
        __syncwarp();
      }
      stream_members<D, KIND, NR, TILE, SELF, false, RT, F32S>(S, rec, nmem, o, kp, worker, grp, G, x, acc, ntile);
    }
    constexpr double SCALE = kscale<KIND>() * (is_inv_r<KIND>() ? 0.5 : 1.0);
#pragma unroll
    for (int t = 0; t < RT; t++)
#pragma unroll
      for (int r = 0; r < NR; r++) S.part[(t * 32 + lane) * NR + r] = acc[t][r];
    __syncwarp();
    if (worker && grp == 0) {
#pragma unroll
      for (int t = 0; t < RT; t++) {
        if (!act[t]) continue;
        const int64_t a = a0 + slot + t * TS;
#pragma unroll
        for (int r = 0; r < NR; r++) {
          double tot = 0.0;
          for (int g = 0; g < G; g++) tot += S.part[(t * 32 + g * TS + slot) * NR + r];
          T.out[(tb + a) * R + r0 + r] = tot * SCALE;
        }
      }
    }
    __syncwarp();
  }
}

// Lane layout per cell: RT targets per lane, TS = ceil(m / RT) lanes per
// target group, G = 32 / TS groups.  RT = 3 is taken when it wastes fewer
// lane-pair slots than RT = 2 (cells of ~13.5 pivots do not tile 32 lanes:
// pair-weighted lane efficiency 0.82 -> 0.90 at the headline).
__device__ __forceinline__ float lane_eff(int m, int rt) {
  const int ts = (m + rt - 1) / rt;
  const int g = ts > 0 ? 32 / ts : 0;
  return g > 0 ? (float)(m * g) / (float)(32 * rt) : 0.f;
}

template <int D, int KIND, int NR, int TILE, bool SELF, bool F32S, class WS>
__device__ __forceinline__ void interact_cell(const LevelTab& T, int64_t c, const int4 dsc, int64_t R, int64_t r0,
                                              const KParams& kp, WS& S, uint32_t& ntile) {
  if constexpr (WS::RTMAX >= 3) {
    const int m = dsc.y;
    if (m <= 96 && lane_eff(m, 3) > lane_eff(m, 2)) {
      interact_cell_rt<D, KIND, NR, TILE, SELF, 3, F32S>(T, c, dsc, R, r0, kp, S, ntile);
      return;
    }
  }
  interact_cell_rt<D, KIND, NR, TILE, SELF, 2, F32S>(T, c, dsc, R, r0, kp, S, ntile);
}

// item descriptors {first target, targets, list begin, list end} (one 16-byte load per work item)
__global__ void make_item_desc(const int64_t* __restrict__ items, int64_t n, const LevelTab* __restrict__ tabs,
                               int4* __restrict__ desc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t it = items[i];
  const int lev = (int)(it >> 40);
  const int64_t c = it & ((1ll << 40) - 1);
  const LevelTab& T = tabs[lev];
  const int64_t tb = T.t_ptr[c];
  desc[i] = make_int4((int)tb, (int)(T.t_ptr[c + 1] - tb), (int)T.l_ptr[c], (int)(T.l_ptr[c] + T.m_cnt[c]));
}

// Persistent kernel: every warp pulls work items (descending pair count) from
// a global counter until the list is exhausted.
template <int D, int KIND, int NR, int TILE, int RT, bool F32S>
__global__ void __launch_bounds__(IT2, NR == 1 ? H2B_MINB : 2) interact_warps(const int64_t* __restrict__ items, const int4* __restrict__ descs,
                                                      int64_t n_items, unsigned long long* __restrict__ counter,
                                                      const LevelTab* __restrict__ tabs, int ntabs, int near_list,
                                                      int64_t R, int64_t r0, KParams kp) {
  using WS = WarpSmem<D, NR, TILE, RT>;  // RT = the largest targets-per-lane used
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LevelTab* tab_s = reinterpret_cast<LevelTab*>(smem_raw);
  const size_t tab_bytes = (sizeof(LevelTab) * ntabs + 127) / 128 * 128;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WS& S = reinterpret_cast<WS*>(smem_raw + tab_bytes)[warp];
  for (int i = threadIdx.x; i < ntabs; i += blockDim.x) tab_s[i] = tabs[i];
  if (lane == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t ntile = 0;
  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= (unsigned long long)n_items) break;
    const int64_t it = items[idx];
    const int4 dsc = descs[idx];
    const int lev = (int)(it >> 40);
    const int64_t c = it & ((1ll << 40) - 1);
    const LevelTab& T = tab_s[lev];
    if (lev == near_list)
      interact_cell<D, KIND, NR, TILE, true, F32S>(T, c, dsc, R, r0, kp, S, ntile);
    else
      interact_cell<D, KIND, NR, TILE, false, F32S>(T, c, dsc, R, r0, kp, S, ntile);
  }
}

// Records of every source list for one RHS chunk: coordinates (static) and
// charges of columns [r0, r0 + NR) (per matvec).  One thread per record.
struct PackTab {
  const double* sc;  // source coords SoA (ld)
  int64_t ld;
  const double* q;   // charges, row stride R
  double2* rec;      // records
  int64_t n;         // records in this list
  int64_t off;       // first global thread of this list
};

template <int D, int NR>
__global__ void pack_records(const PackTab* __restrict__ pt, int nlists, int64_t total, int64_t R, int64_t r0,
                             int coords) {
  constexpr int W = SrcRec<D, NR>::W;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= total) return;
  int l = 0;
  while (l + 1 < nlists && pt[l + 1].off <= g) l++;
  const PackTab T = pt[l];
  const int64_t i = g - T.off;
  double* r = reinterpret_cast<double*>(T.rec + i * W);
  if (coords) {
#pragma unroll
    for (int k = 0; k < D; k++) r[k] = T.sc[k * T.ld + i];
#pragma unroll
    for (int k = D + NR; k < 2 * W; k++) r[k] = 0.0;
  }
#pragma unroll
  for (int q = 0; q < NR; q++) r[D + q] = T.q[i * R + r0 + q];
}

// per-matvec charge pack, one thread per (record, RHS): coalesced reads of the RHS rows and writes of the
// record's charge slots (the thread-per-record form strides 8 * R bytes per lane on both sides)
template <int D, int NR>
__global__ void pack_charges(const PackTab* __restrict__ pt, int nlists, int64_t total, int64_t R, int64_t r0) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= total * NR) return;
  const int64_t e = g / NR;
  const int q = (int)(g - e * NR);
  int l = 0;
  while (l + 1 < nlists && pt[l + 1].off <= e) l++;
  const PackTab& T = pt[l];
  const int64_t i = e - T.off;
  reinterpret_cast<double*>(T.rec + i * SrcRec<D, NR>::W)[D + q] = T.q[i * R + r0 + q];
}

template <int D, int KIND, int NR, int TILE, bool F32S>
void launch_chunk(const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  if (!h.n_items) return;
  const int nl = h.t->depth + 1;  // list id of the leaf near field
  const int ntabs = nl + 1;
  auto* tabs = reinterpret_cast<const LevelTab*>(h.tabs.get());
  const size_t smem = (sizeof(LevelTab) * ntabs + 127) / 128 * 128 +
                      (IT2 / 32) * sizeof(WarpSmem<D, NR, TILE, (NR == 1 ? H2B_RT : 2)>);
  auto kern = interact_warps<D, KIND, NR, TILE, (NR == 1 ? H2B_RT : 2), F32S>;
  // persistent grid = resident CTAs; attribute and occupancy are per device, so they are set on every call
  // (a process may drive several GPUs)
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, nsm = 0, per = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, IT2, smem));
  const int grid = nsm * (per > 0 ? per : 1);
  // pack this chunk's charges into the records
  const auto& pk = NR == 1 ? h.pack1 : h.pack16;
  if (pk.total && !(NR == 1 && R == 1)) {  // one RHS: gather / upward pass already wrote the charges
    if (NR > 1)
      pack_charges<D, NR><<<nblk(pk.total * NR, 256), 256, 0, s>>>(reinterpret_cast<const PackTab*>(pk.tabs.get()),
                                                                   pk.nlists, pk.total, R, r0);
    else
      pack_records<D, NR><<<nblk(pk.total, 256), 256, 0, s>>>(reinterpret_cast<const PackTab*>(pk.tabs.get()),
                                                              pk.nlists, pk.total, R, r0, 0);
    CKL();
  }
  CK(cudaMemsetAsync(h.work_counter.get(), 0, sizeof(unsigned long long), s));
  const int64_t ng = std::min<int64_t>(grid, (h.n_items + IT2 / 32 - 1) / (IT2 / 32));
  kern<<<(unsigned)ng, IT2, smem, s>>>(h.items.get(), reinterpret_cast<const int4*>(h.item_desc.get()), h.n_items,
                                       h.work_counter.get(), tabs, ntabs, nl, R, r0, kp);
  CKL();
}

template <int D, int NR>
void pack_coords_d(const DevH2& h, cudaStream_t s) {
  const auto& pk = NR == 1 ? h.pack1 : h.pack16;
  if (pk.total)
    pack_records<D, NR><<<nblk(pk.total, 256), 256, 0, s>>>(reinterpret_cast<const PackTab*>(pk.tabs.get()),
                                                            pk.nlists, pk.total, 1, 0, 1);
  CKL();
}

// The FP32-seeded M2L path needs every interaction-list r^2 inside
// [2^-100, 2^100].  Admissible cells at level l satisfy diam <= eta * gap
// (geometry.py:147), so r >= 2 hw_l sqrt(d) / eta >= 2 hw_depth sqrt(d) / eta;
// in the shifted frame every term of r^2 is bounded by (4 sqrt(d) half)^2.
// Otherwise (tests scale the geometry by 2^+-100) the cubic FP64-seeded path runs.
inline bool f32seed_ok(const DevH2& h) {
  const DevTree& t = *h.t;
  const double hw = t.half * std::ldexp(1.0, -t.depth);
  const double rmin = 2.0 * hw * std::sqrt((double)t.d) / (t.eta > 0 ? t.eta : 1.0);
  const double rmax = 4.0 * std::sqrt((double)t.d) * t.half;
  return rmin * rmin > std::ldexp(1.0, -100) && rmax * rmax < std::ldexp(1.0, 100);
}

template <int D, int KIND>
void launch_interact2(const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp, cudaStream_t s) {
  if constexpr (is_inv_r<KIND>()) {
    if (f32seed_ok(h)) {
      if (nr == 16) launch_chunk<D, KIND, 16, H2B_TILE16, true>(h, R, r0, kp, s);
      else launch_chunk<D, KIND, 1, H2B_TILE1, true>(h, R, r0, kp, s);
      return;
    }
  }
  if (nr == 16) launch_chunk<D, KIND, 16, H2B_TILE16, false>(h, R, r0, kp, s);
  else launch_chunk<D, KIND, 1, H2B_TILE1, false>(h, R, r0, kp, s);
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
template <int D>
void pack_coords_dim(const DevH2& h, int nr, cudaStream_t s);

}  // namespace h2b
