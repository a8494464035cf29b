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
#include <cub/cub.cuh>

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

// ---------------------------------------------------------------------
// Interaction kernel: one launch for every M2L level and the near field.
//
// Work item = (list kind, cell).  Items are sorted by their pair count
// (largest first) so the 6-7 M2L levels and the leaf near field share one
// grid with a balanced tail.  A CTA owns one target cell: targets live in
// registers, the cell's source list (interaction list: pivot coordinates +
// multipole charges; neighbour list: points + input charges) is streamed
// through shared-memory tiles and read as warp broadcasts.
// ---------------------------------------------------------------------
constexpr int IT2 = 128;
constexpr int MAXMEM = 128;

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
template <int D, int KIND, int NR, int TILE, bool SELF>
__device__ __forceinline__ void interact_cell(const LevelTab& T, int64_t c, int64_t R, int64_t r0, const KParams& kp,
                                              double2* tile, int64_t* pref, int64_t* sbeg, int64_t* wsum,
                                              double* part) {
  constexpr int RT = 2;
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

template <int D, int KIND, int NR, int TILE>
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
    interact_cell<D, KIND, NR, TILE, true>(T, c, R, r0, kp, tile, pref, sbeg, wsum, part);
  else
    interact_cell<D, KIND, NR, TILE, false>(T, c, R, r0, kp, tile, pref, sbeg, wsum, part);
}

template <int D, int KIND>
void launch_interact2(const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp, cudaStream_t s) {
  const int64_t* items = h.items.get();
  const LevelTab* tabs = reinterpret_cast<const LevelTab*>(h.tabs.get());
  unsigned g = (unsigned)h.n_items;
  const int nl = h.t->depth + 1;  // list id of the leaf near field
  if (!g) return;
  switch (nr) {
    case 16: interact2<D, KIND, 16, 64><<<g, IT2, 0, s>>>(items, tabs, nl, R, r0, kp); break;
    case 8: interact2<D, KIND, 8, 128><<<g, IT2, 0, s>>>(items, tabs, nl, R, r0, kp); break;
    case 4: interact2<D, KIND, 4, 256><<<g, IT2, 0, s>>>(items, tabs, nl, R, r0, kp); break;
    case 2: interact2<D, KIND, 2, 512><<<g, IT2, 0, s>>>(items, tabs, nl, R, r0, kp); break;
    default: interact2<D, KIND, 1, 512><<<g, IT2, 0, s>>>(items, tabs, nl, R, r0, kp); break;
  }
  CKL();
}

template <int D>
void interact_all_d(int kind, const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp, cudaStream_t s) {
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

void interact_all(int d, int kind, const DevH2& h, int64_t R, int64_t r0, int nr, const KParams& kp,
                  cudaStream_t s) {
  switch (d) {
    case 1: interact_all_d<1>(kind, h, R, r0, nr, kp, s); break;
    case 2: interact_all_d<2>(kind, h, R, r0, nr, kp, s); break;
    case 3: interact_all_d<3>(kind, h, R, r0, nr, kp, s); break;
    default: interact_all_d<4>(kind, h, R, r0, nr, kp, s); break;
  }
}

// u[perm[i]] = near[i] + P_c u_in(c)   (L2P fused with the scatter back to the caller's order)
__global__ void l2p_scatter(int64_t ncell, const int64_t* __restrict__ t_ptr, const double* __restrict__ pm,
                            const int64_t* __restrict__ pm_off, const int64_t* __restrict__ kin,
                            const int64_t* __restrict__ in_ptr, const double* __restrict__ uin,
                            const double* __restrict__ near, const int64_t* __restrict__ perm,
                            double* __restrict__ u, int64_t R) {
  const int64_t c = blockIdx.x;
  const int64_t tb = t_ptr[c], m = t_ptr[c + 1] - tb;
  const int64_t k = pm ? kin[c] : 0;
  const double* Pc = pm ? pm + pm_off[c] : nullptr;
  const double* uc = pm ? uin + in_ptr[c] * R : nullptr;
  for (int64_t q = threadIdx.x; q < m * R; q += blockDim.x) {
    const int64_t a = q / R, r = q - a * R;
    double v = near[(tb + a) * R + r];
    for (int64_t s2 = 0; s2 < k; s2++) v = fma(Pc[s2 * m + a], uc[s2 * R + r], v);
    u[perm[tb + a] * R + r] = v;
  }
}

// pair counts per work item (the reference's entry counts for S and near blocks)
__global__ void item_costs(int64_t n, int lev, const int64_t* __restrict__ t_ptr, const int64_t* __restrict__ s_ptr,
                           const int64_t* __restrict__ l_ptr, const int64_t* __restrict__ l_idx,
                           unsigned long long* __restrict__ cost, int64_t* __restrict__ item) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  int64_t src = 0;
  for (int64_t q = l_ptr[c]; q < l_ptr[c + 1]; q++) {
    int64_t y = l_idx[q];
    src += s_ptr[y + 1] - s_ptr[y];
  }
  cost[c] = (unsigned long long)((t_ptr[c + 1] - t_ptr[c]) * src);
  item[c] = ((int64_t)lev << 40) | c;
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

// work list: every M2L (level, cell) and every leaf near-field cell, by descending pair count
void build_items(DevH2& h, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth;
  int64_t total = T.lv[L].n;
  for (int l = 2; l <= L; l++) total += T.lv[l].n;
  DBuf<unsigned long long> cost, cost_sorted;
  DBuf<int64_t> item;
  cost.alloc(total);
  cost_sorted.alloc(total);
  item.alloc(total);
  h.items.alloc(total, &h.mem);
  int64_t off = 0;
  for (int l = 2; l <= L; l++) {
    const DevLevel& Lv = T.lv[l];
    const DevH2Level& HL = h.lv[l];
    if (Lv.n)
      item_costs<<<ceil_div(Lv.n, 256), 256, 0, s>>>(Lv.n, l, HL.in_ptr.get(), HL.out_ptrd(), Lv.il_ptr.get(),
                                                     Lv.il_idx.get(), cost.get() + off, item.get() + off);
    CKL();
    off += Lv.n;
  }
  {
    const DevLevel& Lv = T.lv[L];
    item_costs<<<ceil_div(Lv.n, 256), 256, 0, s>>>(Lv.n, L + 1, Lv.t_ptr.get(),
                                                   T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get(), Lv.nb_ptr.get(),
                                                   Lv.nb_idx.get(), cost.get() + off, item.get() + off);
    CKL();
  }
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, cost.get(), cost_sorted.get(), item.get(),
                                               h.items.get(), total, 0, 64, s));
  DBuf<unsigned char> tmp;
  tmp.alloc(bytes);
  CK(cub::DeviceRadixSort::SortPairsDescending(tmp.get(), bytes, cost.get(), cost_sorted.get(), item.get(),
                                               h.items.get(), total, 0, 64, s));
  // drop zero-cost items (cells with no targets or an empty list)
  auto hc = to_host(cost_sorted.get(), total, s);
  int64_t nz = 0;
  while (nz < total && hc[nz] > 0) nz++;
  h.n_items = nz;
}

void build_tabs(DevH2& h, int64_t R, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth;
  std::vector<LevelTab> tabs(L + 2);
  for (int l = 2; l <= L; l++) {
    const DevLevel& Lv = T.lv[l];
    const DevH2Level& HL = h.lv[l];
    LevelTab& t = tabs[l];
    t.tc = HL.tin_c.get();
    t.ld_t = std::max<int64_t>(HL.in_total, 1);
    t.t_ptr = HL.in_ptr.get();
    t.sc = HL.sout_cd();
    t.ld_s = std::max<int64_t>(HL.out_total, 1);
    t.s_ptr = HL.out_ptrd();
    t.q = h.wout[l].get();
    t.l_ptr = Lv.il_ptr.get();
    t.l_idx = Lv.il_idx.get();
    t.out = h.uin[l].get();
  }
  const DevLevel& Lv = T.lv[L];
  LevelTab& t = tabs[L + 1];
  t.tc = T.tsd();
  t.ld_t = T.np;
  t.t_ptr = Lv.t_ptr.get();
  t.sc = T.ssd();
  t.ld_s = T.nq;
  t.s_ptr = T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get();
  t.q = h.w_sorted.get();
  t.l_ptr = Lv.nb_ptr.get();
  t.l_idx = Lv.nb_idx.get();
  t.out = h.near.get();
  h.tabs.alloc(sizeof(LevelTab) * tabs.size(), &h.mem);
  CK(cudaMemcpyAsync(h.tabs.get(), tabs.data(), sizeof(LevelTab) * tabs.size(), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
}

void ensure_scratch(DevH2& h, int64_t R, cudaStream_t s) {
  const DevTree& T = *h.t;
  if (h.scratch_nrhs == R) return;
  h.w_sorted.alloc(T.nq * R, &h.mem);
  h.near.alloc(T.np * R, &h.mem);
  h.wout.clear();
  h.uin.clear();
  h.wout.resize(T.depth + 1);
  h.uin.resize(T.depth + 1);
  for (int l = 2; l <= T.depth; l++) {
    h.wout[l].alloc(std::max<int64_t>(h.lv[l].out_total * R, 1), &h.mem);
    h.uin[l].alloc(std::max<int64_t>(h.lv[l].in_total * R, 1), &h.mem);
  }
  if (!h.items.n) build_items(h, s);
  build_tabs(h, R, s);
  h.scratch_nrhs = R;
}

// RHS widths supported by the interaction kernel
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

void prepare_matvec(DevH2& h, cudaStream_t s) { ensure_scratch(h, 1, s); }

void set_profiling(bool on) { g_profile = on; }
void last_stage_ms(double* ms5) {
  for (int i = 0; i < 5; i++) ms5[i] = g_stage_ms[i];
}

int64_t matvec_launches(const DevH2& h, int64_t nrhs) {
  const int L = h.t->depth;
  std::vector<std::pair<int64_t, int>> ch;
  rhs_chunks(nrhs, ch);
  int64_t nchunk = (int64_t)ch.size();
  if (L < 2) return 1 + nchunk + 1;
  // gather, P2M, M2M x (L-2), interaction x chunks, L2L x (L-2), L2P+scatter
  return 1 + 1 + (L - 2) + nchunk + (L - 2) + 1;
}

void matvec(DevH2& h, const double* w, double* u, int64_t R, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth, d = T.d;
  ensure_scratch(h, R, s);
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
  }
  if (g_profile) CK(cudaEventRecord(ev[1], s));
  // ---- every M2L level + the near field in one launch ----
  for (auto& ch : chunks) interact_all(d, h.kind, h, R, ch.first, ch.second, kp, s);
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
  if (g_profile) CK(cudaEventRecord(ev[3], s));
  // ---- L2P + near field, scattered to the caller's order ----
  {
    const DevLevel& Lv = T.lv[L];
    const bool far = L >= 2;
    const DevH2Level* HL = far ? &h.lv[L] : nullptr;
    l2p_scatter<<<(unsigned)Lv.n, 128, 0, s>>>(Lv.n, Lv.t_ptr.get(), far ? HL->pmat.get() : nullptr,
                                               far ? HL->pm_off.get() : nullptr, far ? HL->kin.get() : nullptr,
                                               far ? HL->in_ptr.get() : nullptr, far ? h.uin[L].get() : nullptr,
                                               h.near.get(), T.t_perm.get(), u, R);
    CKL();
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
