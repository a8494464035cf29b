// interact_sym.cuh — symmetric interaction kernel (one right-hand side).
//
// On the symmetric path (symmetric kernel on shared points, compress.py:229)
// the outgoing pivots of a cell are its incoming ones (s_out = t_in,
// compress.py:254-260), so the coupling blocks satisfy S_{Y,X} = S_{X,Y}^T
// and the near-field blocks K(Y, X) = K(X, Y)^T.  The reference evaluates
// and applies both ordered blocks (compress.py:307-328, matvec.py:161); here
// each unordered cell pair {X, Y} is evaluated once, by the work item of the
// lower cell (Y > X in the engine's Morton order), and applied in both
// directions:
//     u_in^X += S_{X,Y} w_out^Y      (row sums: X's targets)
//     u_in^Y += S_{X,Y}^T w_out^X    (column sums: Y's targets)
// which halves the kernel evaluations (r^2 + rsqrt + Newton) per product.
//
// Work item = (list, cell X): list l in [2, L] is level l's interaction list,
// L + 1 the leaf near field: neighbour leaves Y > X plus X itself, whose
// block K(X, X) is evaluated in both orders with row sums only (r2 == 0 ->
// 0, the punctured diagonal); difference-form r^2.  One warp per item.  X's targets are staged TB at a
// time in the warp's shared memory and broadcast; the "upper" partners'
// source records (contiguous Morton ranges, adjacent ones merged) are spread
// over the lanes, RS records per lane held in registers with their column
// accumulators.  Per (target, lane) the lane evaluates RS pairs:
//     r2  = |x'|^2 + |y'|^2 - 2 x'.y'            (M2L; DADD + 3 DFMA)
//     K   = K(r2)                                 (1/r: FP32 seed, DMUL, DFMA, DMUL)
//     col_s += K q_t ;  p_t += K q_s              (2 DFMA)
// 9 FP64 instructions per unordered pair = 4.5 per applied entry (the
// one-directional kernel, interact.cuh, needs 8).  The TB row partials p_t
// live in registers for the whole chunk and are reduced across the warp once
// per chunk (butterfly reduce-scatter); column sums are flushed after every
// pass.  Both go to the level's u_in (and the near-field buffer) with FP64
// reductions (RED.ADD.F64), so those buffers are zeroed first.
#pragma once
#include <climits>

#include "interact.cuh"

namespace h2b {
namespace {

#ifndef H2B_SYM_RS
#define H2B_SYM_RS 2
#endif
constexpr int SYM_NARROW = 16;  // target chunks of 16 (4 CTAs / SM, 128 registers) unless most pairs sit in items
                                // with more targets: then chunks of 32 (fewer source passes), 3 CTAs / SM
constexpr int SYM_THREADS = 128;
constexpr int SYM_MAXMEM = 256;  // members staged per chunk of a cell's upper list

// Per-list tables of the symmetric kernel (device copy, one per list id).
struct SymTab {
  const double2* rec;  // source records [y_0..y_{D-1}, q] (SrcRec<D, 1>) of this list's points
  const int64_t* ptr;  // record range per cell (targets == sources on the symmetric path)
  const int* m_sb;     // upper member tables: first record of each (merged) member
  const int* m_end;    //   inclusive prefix of member lengths within the cell's segment
  double* out;         // result rows (record index) * R + r0
};

enum SymMode { SYM_M2L = 0, SYM_NEAR = 1 };

template <int D>
struct alignas(16) SymTgt {  // one staged target: M2L a = (-2 x', |x'|^2), near a = x'
  static constexpr int A = D + 1;
  static constexpr int N2 = 2 * ((A + 1 + 1) / 2);  // doubles incl. q, padded to 16 bytes
  double v[N2];
};

#ifndef H2B_SYM_MAP
#define H2B_SYM_MAP 1024
#endif
constexpr int SYM_MAP = H2B_SYM_MAP;  // slots of a source window (record indices staged in shared memory)

template <int D>
struct alignas(16) SymWarp {
  SymTgt<D> tgt[32];
  double2 rbuf[2][32 * H2B_SYM_RS * SrcRec<D, 1>::W];  // source records of the current / next pass (cp.async)
  int pref[SYM_MAXMEM + 1];
  int sbeg[SYM_MAXMEM];
  int map[SYM_MAP];  // window slot -> record index
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// FP64 reduction into global memory.  atomicAdd on a generic pointer compiles to a run-time address-space
// dispatch (QSPC + three code paths, ~25 instructions per call); the level buffers are always global.
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "d"(v) : "memory");
}

template <int D>
__device__ __forceinline__ void load_rec(const double2* rec, int64_t i, double (&y)[D], double& q) {
  constexpr int W = SrcRec<D, 1>::W;
  double v[2 * W];
#pragma unroll
  for (int w = 0; w < W; w++) {
    const double2 u = __ldg(rec + i * W + w);
    v[2 * w] = u.x;
    v[2 * w + 1] = u.y;
  }
#pragma unroll
  for (int k = 0; k < D; k++) y[k] = v[k];
  q = v[D];
}

// K(r2) in the kernel's accumulation units (1/r: "2/r", scaled at the flush)
template <int KIND, int MODE, bool F32S>
__device__ __forceinline__ double sym_kval(double r2, const KParams& kp) {
  if constexpr (is_inv_r<KIND>()) {
    if constexpr (MODE == SYM_NEAR) {
      // near field (plain input charges): FP64 seed + quadratic step; the item's own leaf is among the sources,
      // so r2 == 0 (a point with itself or a duplicate) gives 0, the punctured diagonal
      const bool zero = __double2hiint(r2) == 0;  // r2 == 0 (or subnormal)
      const double r2s = zero ? 1.0 : r2;
      const double y = rsq_approx(r2s);
      const double kv = y * fma(-r2s, y * y, 3.0);
      return zero ? 0.0 : kv;
    } else if constexpr (F32S) {
      const double y = rsq_seed_f32(r2);  // FP32 seed + quadratic step (interact.cuh rsq_seed_f32)
      return y * fma(-r2, y * y, 3.0);
    } else {
      const double y = rsq_approx(r2);  // FP64 seed + cubic step (multipole charges amplify a bias)
      const double e = fma(-r2, y * y, 1.0);
      return y * fma(e, fma(0.75, e, 1.0), 2.0);
    }
  } else {
    return kfast<KIND>(r2, kp);
  }
}

// Sum of the TB (16 or 32) row partials over the warp by a butterfly reduce-scatter: afterwards lane l holds
// the total of target l / (32 / TB).
template <int TB>
__device__ __forceinline__ double warp_reduce_scatter(const double (&p)[TB], int lane) {
  static_assert(TB == 16 || TB == 32, "TB must be 16 or 32");
  double v[TB];
#pragma unroll
  for (int i = 0; i < TB; i++) v[i] = p[i];
#pragma unroll
  for (int half = TB / 2, bit = 16; half >= 1; half /= 2, bit /= 2) {
    const bool hi = lane & bit;
#pragma unroll
    for (int i = 0; i < half; i++) {
      const double send = hi ? v[i] : v[i + half];
      const double keep = hi ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
    }
  }
  double r = v[0];
#pragma unroll
  for (int bit = 32 / TB / 2; bit >= 1; bit /= 2) r += __shfl_xor_sync(0xffffffffu, r, bit);
  return r;
}

// One pair: r^2, K, and both accumulations.
template <int D, int KIND, int MODE, bool F32S, int NV>
__device__ __forceinline__ void sym_pair(const double (&a)[NV], const double (&y)[D], double yy, double qs,
                                         double& col, double& p, const KParams& kp) {
  double r2;
  if constexpr (MODE == SYM_M2L) {
    r2 = a[D] + yy;
#pragma unroll
    for (int k = 0; k < D; k++) r2 = fma(a[k], y[k], r2);
  } else {
    r2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; k++) {
      const double dk = a[k] - y[k];
      r2 = fma(dk, dk, r2);
    }
  }
  const double kv = sym_kval<KIND, MODE, F32S>(r2, kp);
  col = fma(kv, a[D + 1], col);
  p = fma(kv, qs, p);
}

template <int D>
__device__ __forceinline__ void load_tgt(const SymWarp<D>& S, int t, double (&a)[SymTgt<D>::N2]) {
#pragma unroll
  for (int i = 0; i < SymTgt<D>::N2; i += 2) {
    const double2 u = *reinterpret_cast<const double2*>(&S.tgt[t].v[i]);
    a[i] = u.x;
    a[i + 1] = u.y;
  }
}

// One work item on one warp.  Loop nest: member chunks (<= SYM_MAXMEM members, table in shared memory) >
// source windows (<= SYM_MAP records; slot -> record index map expanded in shared memory) > target chunks
// (TB targets staged, padded to an even count with a zero-charge copy) > passes (RS records per lane).
template <int D, int KIND, int RS, int TB, bool F32S, int MODE>
__device__ __forceinline__ void sym_item(const SymTab& T, int4 dsc, int64_t R, int64_t r0, const KParams& kp,
                                         SymWarp<D>& S) {
  constexpr double SCALE = kscale<KIND>() * (is_inv_r<KIND>() ? 0.5 : 1.0);
  constexpr int NV = SymTgt<D>::N2;
  const int lane = threadIdx.x & 31;
  const int tb = dsc.x, m = dsc.y, lb = dsc.z, cnt = dsc.w;
  const double2* rec = T.rec;  // in registers: the cp.async asm statements would force reloads from T
  double* out = T.out;
  double o[D];  // frame origin: the item's first target
  {
    double q;
    load_rec<D>(rec, tb, o, q);
  }
  // virtual member list: near field = [the leaf itself (row sums only: both orders of each pair inside the
  // block are evaluated), upper neighbours]; M2L = [upper interaction-list cells]
  constexpr int SELF0 = MODE == SYM_NEAR ? 1 : 0;
  const int vc = cnt + SELF0;
  for (int v0 = 0; v0 < vc; v0 += SYM_MAXMEM) {
    const int nmem = vc - v0 < SYM_MAXMEM ? vc - v0 : SYM_MAXMEM;
    __syncwarp();
    {
      const int r0m = v0 - SELF0;  // real member index of virtual index v0
      const int base = r0m <= 0 ? 0 : T.m_end[lb + r0m - 1];
      const int selfn = (SELF0 && v0 == 0) ? m : 0;
      for (int i = lane; i < nmem; i += 32) {
        const int r = r0m + i;
        if (r < 0) {
          S.sbeg[i] = -(tb + 1);  // row-only member: the item's own leaf
          S.pref[i + 1] = m;
        } else {
          S.sbeg[i] = T.m_sb[lb + r];
          S.pref[i + 1] = selfn + T.m_end[lb + r] - base;
        }
      }
      if (lane == 0) S.pref[0] = 0;
    }
    __syncwarp();
    const int total = S.pref[nmem];
    for (int w0 = 0; w0 < total; w0 += SYM_MAP) {
      const int wn = total - w0 < SYM_MAP ? total - w0 : SYM_MAP;
      __syncwarp();
      for (int i = lane; i < nmem; i += 32) {  // expand the members overlapping the window
        const int pa = S.pref[i], pe = S.pref[i + 1];
        const int a = pa > w0 ? pa : w0, e = pe < w0 + wn ? pe : w0 + wn;
        const int sg = S.sbeg[i];
        if (sg >= 0) {
          for (int j = a; j < e; j++) S.map[j - w0] = sg + (j - pa);
        } else {  // row-only records are stored as -(index + 1)
          for (int j = a; j < e; j++) S.map[j - w0] = sg - (j - pa);
        }
      }
      for (int tc0 = 0; tc0 < m; tc0 += TB) {
        const int tcnt = m - tc0 < TB ? m - tc0 : TB;
        const int tpad = (tcnt + 1) & ~1;
        __syncwarp();
        if (lane < tpad) {  // stage this chunk's targets (an odd count gets a zero-charge copy of the first)
          double x[D], q;
          load_rec<D>(rec, tb + tc0 + (lane < tcnt ? lane : 0), x, q);
          double* v = S.tgt[lane].v;
          double n2 = 0.0;
#pragma unroll
          for (int k = 0; k < D; k++) {
            const double dk = x[k] - o[k];
            n2 = fma(dk, dk, n2);
            v[k] = MODE == SYM_M2L ? -2.0 * dk : dk;
          }
          v[D] = n2;
          v[D + 1] = lane < tcnt ? q : 0.0;
        }
        __syncwarp();
        double p[TB];
#pragma unroll
        for (int t = 0; t < TB; t++) p[t] = 0.0;
        // passes of 32 RS slots; each lane copies its own slots' records for the next pass (cp.async) while the
        // current one computes, and reads back only what it copied itself (no cross-lane synchronisation)
        constexpr int W = SrcRec<D, 1>::W;
        int gnext[RS];
        auto issue = [&](int pb, int buf) {
#pragma unroll
          for (int s = 0; s < RS; s++) {
            const int j = pb + lane + 32 * s;
            const int g0 = S.map[j < wn ? j : pb];  // dummy slot: a copy of the pass's first source
            gnext[s] = j < wn ? g0 : INT_MIN;
            const int g = g0 >= 0 ? g0 : -g0 - 1;
#pragma unroll
            for (int w = 0; w < W; w++) cp_async16(&S.rbuf[buf][(lane + 32 * s) * W + w], rec + (int64_t)g * W + w);
          }
          cp_async_commit();
        };
        issue(0, 0);
        int pi = 0;
        for (int pb = 0; pb < wn; pb += 32 * RS, pi ^= 1) {
          int gidx[RS];
#pragma unroll
          for (int s = 0; s < RS; s++) gidx[s] = gnext[s];
          if (pb + 32 * RS < wn) {
            issue(pb + 32 * RS, pi ^ 1);
            cp_async_wait<1>();
          } else {
            cp_async_wait<0>();
          }
          double y[RS][D], yy[RS], qs[RS], col[RS];
#pragma unroll
          for (int s = 0; s < RS; s++) {
            double v[2 * W];
#pragma unroll
            for (int w = 0; w < W; w++) {
              const double2 u = S.rbuf[pi][(lane + 32 * s) * W + w];
              v[2 * w] = u.x;
              v[2 * w + 1] = u.y;
            }
            double n2 = 0.0;
#pragma unroll
            for (int k = 0; k < D; k++) {
              y[s][k] = v[k] - o[k];
              n2 = fma(y[s][k], y[s][k], n2);
            }
            yy[s] = n2;
            qs[s] = gidx[s] != INT_MIN ? v[D] : 0.0;
            col[s] = 0.0;
          }
#pragma unroll
          for (int t = 0; t < TB; t += 2) {
            if (t >= tpad) break;
            double a0[NV], a1[NV];
            load_tgt<D>(S, t, a0);
            load_tgt<D>(S, t + 1, a1);
#pragma unroll
            for (int s = 0; s < RS; s++) sym_pair<D, KIND, MODE, F32S, NV>(a0, y[s], yy[s], qs[s], col[s], p[t], kp);
#pragma unroll
            for (int s = 0; s < RS; s++)
              sym_pair<D, KIND, MODE, F32S, NV>(a1, y[s], yy[s], qs[s], col[s], p[t + 1], kp);
          }
#pragma unroll
          for (int s = 0; s < RS; s++)
            if (gidx[s] >= 0) red_add_f64(out + (int64_t)gidx[s] * R + r0, col[s] * SCALE);
        }
        const double tot = warp_reduce_scatter<TB>(p, lane);
        constexpr int LPT = 32 / TB;  // lanes per target after the reduce-scatter
        const int t = lane / LPT;
        if (lane % LPT == 0 && t < tcnt) red_add_f64(out + (int64_t)(tb + tc0 + t) * R + r0, tot * SCALE);
      }
    }
  }
}

// Persistent kernel: warps pull (list, cell) items by descending pair count.
template <int D, int KIND, int RS, int TB, int MINB, bool F32S>
__global__ void __launch_bounds__(SYM_THREADS, MINB)
    interact_sym(const int64_t* __restrict__ items, const int4* __restrict__ descs, int64_t n_items,
                 unsigned long long* __restrict__ counter, const SymTab* __restrict__ tabs, int ntabs, int near_list,
                 int64_t R, int64_t r0, KParams kp) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SymTab* tab_s = reinterpret_cast<SymTab*>(smem_raw);
  const size_t tab_bytes = (sizeof(SymTab) * ntabs + 127) / 128 * 128;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < ntabs; i += blockDim.x) tab_s[i] = tabs[i];
  __syncthreads();
  SymWarp<D>& S = reinterpret_cast<SymWarp<D>*>(smem_raw + tab_bytes)[warp];
  for (;;) {
    unsigned long long idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1ull);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= (unsigned long long)n_items) break;
    const int lst = (int)(items[idx] >> 40);
    const int4 dsc = descs[idx];
    const SymTab& T = tab_s[lst];
    if (lst == near_list)
      sym_item<D, KIND, RS, TB, F32S, SYM_NEAR>(T, dsc, R, r0, kp, S);
    else
      sym_item<D, KIND, RS, TB, F32S, SYM_M2L>(T, dsc, R, r0, kp, S);
  }
}

template <int D, int KIND, int TB, int MINB, bool F32S>
void launch_sym_width(const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  if (!h.n_sym_items) return;
  const int L = h.t->depth;
  auto kern = interact_sym<D, KIND, H2B_SYM_RS, TB, MINB, F32S>;
  int dev = 0, nsm = 0, per = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int ntabs = L + 2;
  const size_t smem = (sizeof(SymTab) * ntabs + 127) / 128 * 128 + (SYM_THREADS / 32) * sizeof(SymWarp<D>);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, SYM_THREADS, smem));
  const int64_t grid = std::min<int64_t>((int64_t)nsm * std::max(per, 1),
                                         (h.n_sym_items + SYM_THREADS / 32 - 1) / (SYM_THREADS / 32));
  CK(cudaMemsetAsync(h.work_counter.get(), 0, sizeof(unsigned long long), s));
  kern<<<(unsigned)grid, SYM_THREADS, smem, s>>>(h.sym_items.get(), reinterpret_cast<const int4*>(h.sym_desc.get()),
                                                 h.n_sym_items, h.work_counter.get(),
                                                 reinterpret_cast<const SymTab*>(h.sym_tabs.get()), ntabs, L + 1,
                                                 R, r0, kp);
  CKL();
}

template <int D, int KIND, bool F32S>
void launch_sym(const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  // one RHS of a wider product: pack this column's charges into the records (the gather / upward pass wrote
  // them already when R == 1)
  const auto& pk = h.pack1;
  if (pk.total && R != 1) {
    pack_records<D, 1><<<nblk(pk.total, 256), 256, 0, s>>>(reinterpret_cast<const PackTab*>(pk.tabs.get()),
                                                           pk.nlists, pk.total, R, r0, 0);
    CKL();
  }
#ifndef H2B_SYM_FORCE
#define H2B_SYM_FORCE 0  // tuning builds: 16 or 32 forces the chunk width
#endif
  if (H2B_SYM_FORCE == 32 || (H2B_SYM_FORCE == 0 && h.sym_wide))
    launch_sym_width<D, KIND, 32, 3, F32S>(h, R, r0, kp, s);
  else
    launch_sym_width<D, KIND, 16, 4, F32S>(h, R, r0, kp, s);
}

template <int D, int KIND>
void launch_sym_kind(const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  if constexpr (is_inv_r<KIND>()) {
    if (f32seed_ok(h)) {
      launch_sym<D, KIND, true>(h, R, r0, kp, s);
      return;
    }
  }
  launch_sym<D, KIND, false>(h, R, r0, kp, s);
}

template <int D>
void interact_sym_d_impl(int kind, const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  switch (kind) {
    case COULOMB: launch_sym_kind<D, COULOMB>(h, R, r0, kp, s); break;
    case LAPLACE: launch_sym_kind<D, LAPLACE>(h, R, r0, kp, s); break;
    case GAUSSIAN: launch_sym_kind<D, GAUSSIAN>(h, R, r0, kp, s); break;
    case GAUSSIAN_SCALED: launch_sym_kind<D, GAUSSIAN_SCALED>(h, R, r0, kp, s); break;
    case MATERN: launch_sym_kind<D, MATERN>(h, R, r0, kp, s); break;
    case LOG: launch_sym_kind<D, LOG>(h, R, r0, kp, s); break;
    case REG_INVERSE: launch_sym_kind<D, REG_INVERSE>(h, R, r0, kp, s); break;
    default: launch_sym_kind<D, REG_LOG>(h, R, r0, kp, s); break;
  }
}

}  // namespace

template <int D>
void interact_sym_d(int kind, const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s);

}  // namespace h2b
