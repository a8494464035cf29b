// transfer.cuh — P2M / M2M / L2L / L2P (matvec.py:169 h2_matvec_reference, passes 1, 2, 4 and 5) on compact
// interpolation operators.
//
// The reference pins the pivot rows of every interpolator to exact identity rows (aca.py:297 row_interpolator,
// :311 col_interpolator; nnca.cu writes the same 1.0 / 0.0 pattern).  A cell's operator (nr x k, nr = its points
// or its children's stacked pivots) therefore has k rows that only copy a value.  The transfer passes are
// HBM-bound on the operator bytes, so the matvec keeps a compact copy without those rows:
//   * piv_pos[p]      row position (in the level's row space: child-level pivot array or sorted points) of
//                     the identity row of pivot p, -1 when the cell is kept dense (no exact identity row found)
//   * g_pos / g_owner the other ("general") rows, cell after cell, g_ptr[c] .. g_ptr[c + 1]
//   * op_dn[s * g + j], op_up[j * k + s]   the g x k general block, row-fastest (downward: one thread per
//                     general row) and column-fastest (upward: one thread per pivot)
// upward:   w_out[s] = x[piv_pos[s]] + sum_j op_up[j * k + s] x[g_pos[j]]
// downward: u[g_pos[j]] (+)= sum_s op_dn[s * g + j] u_in[s];   u[piv_pos[s]] (+)= u_in[s]
// Identity rows contribute exact products (1.0 * x, 0.0 * x), so only the summation order differs from the
// dense form.  At the headline (sphere, N = 2^20) the general blocks hold well under half of the dense bytes.
#pragma once
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include "engine.cuh"

namespace h2b {
namespace {

// one thread per cell writes its owner id over its range
__global__ void fill_owner(int64_t ncell, const int64_t* __restrict__ ptr, int* __restrict__ owner) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= ncell) return;
  for (int64_t p = ptr[c]; p < ptr[c + 1]; p++) owner[p] = (int)c;
}

// One warp per cell: tag every row (identity row of column s / general), pick the first identity row of every
// column as its pivot row, count the general rows.  rowtag lives in the level's row space (cells own disjoint
// row ranges) and ends as 1 = general, 0 = pivot row.
__global__ void classify_rows(int64_t n, const int64_t* __restrict__ ptr, const int64_t* __restrict__ nrow,
                              const double* __restrict__ mat, const int64_t* __restrict__ mat_off,
                              const int64_t* __restrict__ base_ptr, const int64_t* __restrict__ base_map,
                              int* __restrict__ rowtag, int* __restrict__ piv_pos, int64_t* __restrict__ g_cnt,
                              int64_t* __restrict__ op_cnt) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= n) return;
  const int64_t p0 = ptr[c];
  const int k = (int)(ptr[c + 1] - p0);
  const int nr = (int)nrow[c];
  const double* M = mat + mat_off[c];
  const int64_t base = base_ptr[base_map ? base_map[c] : c];
  for (int i = lane; i < nr; i += 32) {
    int tag = -1;
    bool ok = true;
    for (int s = 0; s < k; s++) {
      const double v = M[(int64_t)s * nr + i];
      if (v == 1.0 && tag < 0) tag = s;
      else if (v != 0.0) ok = false;
    }
    rowtag[base + i] = ok ? tag : -1;
  }
  __syncwarp();
  bool all = true;
  for (int s0 = 0; s0 < k; s0 += 32) {
    const int s = s0 + lane;
    int found = -1;
    if (s < k) {
      for (int i = 0; i < nr; i++)
        if (rowtag[base + i] == s) {
          found = i;
          break;
        }
      piv_pos[p0 + s] = found >= 0 ? (int)(base + found) : -1;
    }
    all = __all_sync(0xffffffffu, s >= k || found >= 0) && all;
  }
  if (!all)
    for (int s = lane; s < k; s += 32) piv_pos[p0 + s] = -1;
  __syncwarp();
  int cnt = 0;
  for (int i0 = 0; i0 < nr; i0 += 32) {
    const int i = i0 + lane;
    bool gen = false;
    if (i < nr) {
      const int tag = rowtag[base + i];
      gen = !(all && tag >= 0 && piv_pos[p0 + tag] == (int)(base + i));
      rowtag[base + i] = gen ? 1 : 0;
    }
    cnt += __popc(__ballot_sync(0xffffffffu, gen));
  }
  if (lane == 0) {
    g_cnt[c] = cnt;
    op_cnt[c] = (int64_t)cnt * k;
  }
}

// One warp per cell: general rows in row order, their positions / owner, and the g x k block in both layouts.
__global__ void fill_compact(int64_t n, const int64_t* __restrict__ ptr, const int64_t* __restrict__ nrow,
                             const double* __restrict__ mat, const int64_t* __restrict__ mat_off,
                             const int64_t* __restrict__ base_ptr, const int64_t* __restrict__ base_map,
                             const int* __restrict__ rowtag, const int64_t* __restrict__ g_ptr,
                             const int64_t* __restrict__ op_off, int* __restrict__ g_pos, int* __restrict__ g_owner,
                             double* __restrict__ op_dn, double* __restrict__ op_up) {
  const int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= n) return;
  const int k = (int)(ptr[c + 1] - ptr[c]);
  const int nr = (int)nrow[c];
  const double* M = mat + mat_off[c];
  const int64_t base = base_ptr[base_map ? base_map[c] : c];
  const int64_t gb = g_ptr[c];
  const int g = (int)(g_ptr[c + 1] - gb);
  double* dn = op_dn ? op_dn + op_off[c] : nullptr;
  double* up = op_up ? op_up + op_off[c] : nullptr;
  int run = 0;
  for (int i0 = 0; i0 < nr; i0 += 32) {
    const int i = i0 + lane;
    const bool gen = i < nr && rowtag[base + i] != 0;
    const unsigned b = __ballot_sync(0xffffffffu, gen);
    if (gen) {
      const int j = run + __popc(b & ((1u << lane) - 1u));
      g_pos[gb + j] = (int)(base + i);
      g_owner[gb + j] = (int)c;
      for (int s = 0; s < k; s++) {
        const double v = M[(int64_t)s * nr + i];
        if (dn) dn[(int64_t)s * g + j] = v;
        if (up) up[(int64_t)j * k + s] = v;
      }
    }
    run += __popc(b);
  }
}

inline void exclusive_scan_n1(const int64_t* in_n, int64_t* out_n1, int64_t n, cudaStream_t s) {
  // out has n + 1 entries; in is read as n + 1 entries whose last one is ignored by the exclusive sum
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in_n, out_n1, n + 1, s));
  DBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(bytes, 1));
  CK(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, in_n, out_n1, n + 1, s));
}

// lanes per output row: enough rows in flight, short per-lane chains
inline int lane_group(int64_t rows, int64_t chain) {
  int sg = 1;
  while (sg < 16 && (chain / sg > 24 || rows * sg < 148 * 1024)) {
    if (chain / (2 * sg) < 4) break;
    sg *= 2;
  }
  return sg;
}

// Compact operators of one level and side.  ptr: pivot prefix (n + 1); nrow / mat / mat_off: the dense
// interpolators; rows of cell c start at base_ptr[base_map ? base_map[c] : c] of a row space of `rowspace` rows.
inline void build_compact(CompactOps& C, int64_t n, int64_t npiv, const int64_t* ptr, const int64_t* nrow,
                          const double* mat, const int64_t* mat_off, const int64_t* base_ptr,
                          const int64_t* base_map, int64_t rowspace, bool want_dn, bool want_up, MemStats* ms,
                          cudaStream_t s) {
  if (rowspace >= ((int64_t)1 << 31)) throw std::invalid_argument("more than 2^31 rows in a transfer level");
  DBuf<int> rowtag;
  DBuf<int64_t> g_cnt, op_cnt;
  rowtag.alloc(std::max<int64_t>(rowspace, 1));
  g_cnt.alloc(n + 1);
  op_cnt.alloc(n + 1);
  C.piv_pos.alloc(std::max<int64_t>(npiv, 1), ms);
  C.g_ptr.alloc(n + 1, ms);
  C.op_off.alloc(n + 1, ms);
  if (n)
    classify_rows<<<nblk(n * 32, 256), 256, 0, s>>>(n, ptr, nrow, mat, mat_off, base_ptr, base_map, rowtag.get(),
                                                   C.piv_pos.get(), g_cnt.get(), op_cnt.get());
  CKL();
  exclusive_scan_n1(g_cnt.get(), C.g_ptr.get(), n, s);
  exclusive_scan_n1(op_cnt.get(), C.op_off.get(), n, s);
  C.g_total = read_one(C.g_ptr.get() + n, s);
  C.op_total = read_one(C.op_off.get() + n, s);
  C.g_pos.alloc(std::max<int64_t>(C.g_total, 1), ms);
  C.g_owner.alloc(std::max<int64_t>(C.g_total, 1), ms);
  if (want_dn) C.op_dn.alloc(std::max<int64_t>(C.op_total, 1), ms);
  if (want_up) C.op_up.alloc(std::max<int64_t>(C.op_total, 1), ms);
  if (n)
    fill_compact<<<nblk(n * 32, 256), 256, 0, s>>>(n, ptr, nrow, mat, mat_off, base_ptr, base_map, rowtag.get(),
                                                  C.g_ptr.get(), C.op_off.get(), C.g_pos.get(), C.g_owner.get(),
                                                  want_dn ? C.op_dn.get() : nullptr,
                                                  want_up ? C.op_up.get() : nullptr);
  CKL();
  const int64_t g_avg = n ? C.g_total / n : 0, k_avg = n ? npiv / n : 0;
  C.sg_up = lane_group(npiv, g_avg);
  C.sg_dn = C.g_total < 148 * 1024 ? lane_group(C.g_total, k_avg) : 1;
  CK(cudaStreamSynchronize(s));  // the temporaries above are released on return
  if (getenv("H2B_SETUP_VERBOSE"))
    fprintf(stderr, "[h2b] compact transfers: %lld cells, %lld pivots, %lld general rows of %lld, %.1f MB per layout, lanes up %d down %d\n",
            (long long)n, (long long)npiv, (long long)C.g_total, (long long)rowspace, 8e-6 * (double)C.op_total,
            C.sg_up, C.sg_dn);
}

// RB consecutive doubles of a right-hand-side row: 16-byte loads when every row start is even
template <int RB>
__device__ __forceinline__ void load_rhs(const double* __restrict__ p, bool vec, int64_t r0, int64_t R, double (&v)[RB]) {
  if (RB % 2 == 0 && vec) {
    const double2* p2 = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int i = 0; i < RB / 2; i++) {
      const double2 t = p2[i];
      v[2 * i] = t.x;
      v[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int r = 0; r < RB; r++) v[r] = (RB == 1 || r0 + r < R) ? p[r] : 0.0;
  }
}

// upward (P2M / M2M): thread = (pivot p, block of RB right-hand sides, lane sub of SG).  RB = 1 serves R < 8
// (one thread per (pivot, RHS)) and also writes the charge slot of the pivot's source record when recq is set
// (one RHS: no separate pack pass).  Multi-RHS: each operator entry read once feeds RB accumulators.
template <int SG, int RB>
__global__ void up_compact(int64_t nout, const int* __restrict__ owner, const int64_t* __restrict__ out_ptr,
                           const int* __restrict__ piv_pos, const int64_t* __restrict__ g_ptr,
                           const int* __restrict__ g_pos, const double* __restrict__ op_up,
                           const int64_t* __restrict__ op_off, const double* __restrict__ x, double* __restrict__ y,
                           int64_t R, double* __restrict__ recq, int rs, double* __restrict__ zero) {
  const int64_t nrb = (R + RB - 1) / RB;
  const int64_t qq = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t q = qq / SG;
  const int sub = (int)(qq % SG);
  const bool ok = q < nout * nrb;
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; r++) acc[r] = 0.0;
  int64_t p = 0, r0 = 0;
  if (ok) {
    p = q / nrb;
    r0 = (q - p * nrb) * RB;
    const int c = owner[p];
    const int64_t o0 = out_ptr[c], sidx = p - o0, k = out_ptr[c + 1] - o0;
    const int64_t gb = g_ptr[c];
    const int g = (int)(g_ptr[c + 1] - gb);
    const double* As = op_up + op_off[c] + sidx;
    const int* gp = g_pos + gb;
    const double* xr = x + r0;
    const bool vec = (R % 2 == 0) && r0 + RB <= R;
    for (int j = sub; j < g; j += SG) {
      const double a = As[(int64_t)j * k];
      double xv[RB];
      load_rhs<RB>(xr + (int64_t)gp[j] * R, vec, r0, R, xv);
#pragma unroll
      for (int r = 0; r < RB; r++) acc[r] = fma(a, xv[r], acc[r]);
    }
    if (sub == 0) {
      const int pp = piv_pos[p];
      if (pp >= 0) {
        double xv[RB];
        load_rhs<RB>(xr + (int64_t)pp * R, vec, r0, R, xv);
#pragma unroll
        for (int r = 0; r < RB; r++) acc[r] += xv[r];
      }
    }
  }
  if constexpr (SG > 1) {
#pragma unroll
    for (int r = 0; r < RB; r++)
#pragma unroll
      for (int o = SG / 2; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
  }
  if (ok && sub == 0) {
#pragma unroll
    for (int r = 0; r < RB; r++)
      if (RB == 1 || r0 + r < R) y[p * R + r0 + r] = acc[r];
    if (RB == 1 && recq) recq[q * rs] = acc[0];
    // symmetric one-RHS product: the interaction kernel accumulates into this level's u_in with reductions, so
    // the buffer (one entry per pivot, like y) is cleared here instead of by a memset launch per level
    if (RB == 1 && zero) zero[q] = 0.0;
  }
}

// downward (L2L, and L2P when LEAF): the first gen_threads threads own (general row, RHS block, lane), the rest
// (pivot, RHS block).  L2L accumulates into the child level's u_in (already holding its M2L sums); L2P adds the
// near-field sum and scatters to the caller's order (every target is exactly one general or pivot row).
template <int SG, int RB, bool LEAF>
__global__ void down_compact(int64_t g_total, int64_t npiv, const int* __restrict__ g_owner,
                             const int64_t* __restrict__ g_ptr, const int* __restrict__ g_pos,
                             const int* __restrict__ piv_pos, const int64_t* __restrict__ in_ptr,
                             const double* __restrict__ op_dn, const int64_t* __restrict__ op_off,
                             const double* __restrict__ uin, double* __restrict__ dst,
                             const double* __restrict__ near, const int64_t* __restrict__ perm, int64_t R,
                             int64_t gen_threads) {
  const int64_t nrb = (R + RB - 1) / RB;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; r++) acc[r] = 0.0;
  int64_t pos = -1, r0 = 0;
  bool lead = false;
  if (tid < gen_threads) {  // gen_threads is a multiple of the block size: no warp straddles the two parts
    const int64_t q = tid / SG;
    const int sub = (int)(tid % SG);
    const bool ok = q < g_total * nrb;
    if (ok) {
      const int64_t gq = q / nrb;
      r0 = (q - gq * nrb) * RB;
      const int c = g_owner[gq];
      const int64_t gb = g_ptr[c], g = g_ptr[c + 1] - gb, i0 = in_ptr[c];
      const int k = (int)(in_ptr[c + 1] - i0);
      const double* A = op_dn + op_off[c] + (gq - gb);
      const double* uc = uin + i0 * R + r0;
      const bool vec = (R % 2 == 0) && r0 + RB <= R;
      for (int t = sub; t < k; t += SG) {
        const double a = A[(int64_t)t * g];
        double uv[RB];
        load_rhs<RB>(uc + (int64_t)t * R, vec, r0, R, uv);
#pragma unroll
        for (int r = 0; r < RB; r++) acc[r] = fma(a, uv[r], acc[r]);
      }
      pos = g_pos[gq];
    }
    if constexpr (SG > 1) {
#pragma unroll
      for (int r = 0; r < RB; r++)
#pragma unroll
        for (int o = SG / 2; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    }
    lead = ok && sub == 0;
  } else {
    const int64_t q = tid - gen_threads;
    if (q < npiv * nrb) {
      const int64_t p = q / nrb;
      r0 = (q - p * nrb) * RB;
      const int pp = piv_pos[p];
      if (pp >= 0) {
        const bool vec = (R % 2 == 0) && r0 + RB <= R;
        load_rhs<RB>(uin + p * R + r0, vec, r0, R, acc);
        pos = pp;
        lead = true;
      }
    }
  }
  if (!lead) return;
  if constexpr (LEAF) {
    const int64_t src = pos * R + r0, out = perm[pos] * R + r0;
#pragma unroll
    for (int r = 0; r < RB; r++)
      if (RB == 1 || r0 + r < R) dst[out + r] = near[src + r] + acc[r];
  } else {
    const int64_t out = pos * R + r0;
#pragma unroll
    for (int r = 0; r < RB; r++)
      if (RB == 1 || r0 + r < R) dst[out + r] += acc[r];
  }
}

// trees without a far field (depth < 2): the product is the near-field sum in the caller's order
__global__ void scatter_near(int64_t n, const double* __restrict__ near, const int64_t* __restrict__ perm,
                             double* __restrict__ u, int64_t R) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * R) return;
  const int64_t p = i / R, r = i - p * R;
  u[perm[p] * R + r] = near[i];
}

constexpr int kTransferRB = 8;  // RHS block of the multi-RHS (R >= 8) passes (measured at c4: 8 beats 4 and 16)

inline void launch_up(const CompactOps& C, int64_t nout, const int* owner, const int64_t* out_ptr, const double* x,
                      double* y, int64_t R, cudaStream_t s, double* recq, int rs, double* zero = nullptr) {
  if (R >= 8) {
    const int64_t thr = std::max<int64_t>(nout * ((R + kTransferRB - 1) / kTransferRB), 1);
    up_compact<1, kTransferRB><<<nblk(thr, 256), 256, 0, s>>>(nout, owner, out_ptr, C.piv_pos.get(), C.g_ptr.get(),
                                                              C.g_pos.get(), C.op_up.get(), C.op_off.get(), x, y, R,
                                                              nullptr, 0, nullptr);
    CKL();
    return;
  }
  const int64_t thr = std::max<int64_t>(nout * R, 1) * C.sg_up;
#define H2B_UP(G)                                                                                                 \
  up_compact<G, 1><<<nblk(thr, 256), 256, 0, s>>>(nout, owner, out_ptr, C.piv_pos.get(), C.g_ptr.get(),          \
                                                  C.g_pos.get(), C.op_up.get(), C.op_off.get(), x, y, R, recq, rs, \
                                                  zero)
  switch (C.sg_up) {
    case 1: H2B_UP(1); break;
    case 2: H2B_UP(2); break;
    case 4: H2B_UP(4); break;
    case 8: H2B_UP(8); break;
    default: H2B_UP(16); break;
  }
#undef H2B_UP
  CKL();
}

template <bool LEAF>
inline void launch_down(const CompactOps& C, int64_t npiv, const int64_t* in_ptr, const double* uin, double* dst,
                        const double* near, const int64_t* perm, int64_t R, cudaStream_t s) {
  const int rb = R >= 8 ? kTransferRB : 1;
  const int sg = R >= 8 ? 1 : C.sg_dn;
  const int64_t nrb = (R + rb - 1) / rb;
  const int64_t gen_threads = (int64_t)nblk(C.g_total * nrb * sg, 256) * 256;
  const unsigned blocks = (unsigned)(gen_threads / 256) + nblk(npiv * nrb, 256);
#define H2B_DN(G, B)                                                                                             \
  down_compact<G, B, LEAF><<<blocks, 256, 0, s>>>(C.g_total, npiv, C.g_owner.get(), C.g_ptr.get(), C.g_pos.get(), \
                                                  C.piv_pos.get(), in_ptr, C.op_dn.get(), C.op_off.get(), uin,    \
                                                  dst, near, perm, R, gen_threads)
  if (R >= 8) H2B_DN(1, kTransferRB);
  else
    switch (sg) {
      case 1: H2B_DN(1, 1); break;
      case 2: H2B_DN(2, 1); break;
      case 4: H2B_DN(4, 1); break;
      case 8: H2B_DN(8, 1); break;
      default: H2B_DN(16, 1); break;
    }
#undef H2B_DN
  CKL();
}

}  // namespace
}  // namespace h2b
