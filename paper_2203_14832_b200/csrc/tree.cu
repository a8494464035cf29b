// tree.cu — GPU uniform 2^d tree build (geometry.py:230 build_tree) and
// neighbour / interaction lists (geometry.py:322 _annotate_level).
//
// Bit-exactness: a point's cell at every level comes from the reference's
// own recurrence  bin <- 2*bin + (p > lo0 + (bin + 0.5) * (2*width))  with
// the same two roundings (__dmul_rn then __dadd_rn), so leaf membership is
// identical.  All levels' bins are packed into one 64-bit Morton code per
// point; one radix sort then gives every level's occupancy as runs of code
// prefixes, and the depth is chosen by the reference's stopping rule.
// Lists use the reference's closed-form admissibility test with the same
// roundings (its np.dot is a sequential fused accumulation).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "engine.cuh"

namespace h2b {

namespace {

constexpr double WIDTH_UNDERFLOW = 0x1p-50;

__global__ void bbox_partial(const double* __restrict__ pts, int64_t n, int d, double* lo, double* hi) {
  __shared__ double slo[H2B_MAXD][256];
  __shared__ double shi[H2B_MAXD][256];
  double l[H2B_MAXD], h[H2B_MAXD];
  for (int k = 0; k < d; k++) {
    l[k] = INFINITY;
    h[k] = -INFINITY;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < d; k++) {
      double v = pts[i * d + k];
      l[k] = fmin(l[k], v);
      h[k] = fmax(h[k], v);
    }
  for (int k = 0; k < d; k++) {
    slo[k][threadIdx.x] = l[k];
    shi[k][threadIdx.x] = h[k];
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < d; k++) {
        slo[k][threadIdx.x] = fmin(slo[k][threadIdx.x], slo[k][threadIdx.x + s]);
        shi[k][threadIdx.x] = fmax(shi[k][threadIdx.x], shi[k][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < d; k++) {
      lo[blockIdx.x * d + k] = slo[k][0];
      hi[blockIdx.x * d + k] = shi[k][0];
    }
}

struct BinParams {
  double lo0[H2B_MAXD];
  double w2[64];  // 2 * (half * 2^-l): width of the level-l cell being split
};

// geometry.py:275-279 iterated Lmax times; code packs dim 0 as the most
// significant bit of every level group (== itertools.product child order).
template <int D>
__global__ void morton_codes(const double* __restrict__ pts, int64_t n, int Lmax, BinParams bp,
                             unsigned long long* __restrict__ code, int64_t* __restrict__ idx) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double p[D];
  long long bin[D];
#pragma unroll
  for (int k = 0; k < D; k++) {
    p[k] = pts[i * D + k];
    bin[k] = 0;
  }
  unsigned long long c = 0;
  for (int l = 0; l < Lmax; l++) {
    double w2 = bp.w2[l];
#pragma unroll
    for (int k = 0; k < D; k++) {
      double ctr = __dadd_rn(bp.lo0[k], __dmul_rn((double)bin[k] + 0.5, w2));
      int bit = p[k] > ctr ? 1 : 0;
      bin[k] = 2 * bin[k] + bit;
      c = (c << 1) | (unsigned long long)bit;
    }
  }
  code[i] = c;
  idx[i] = i;
}

__global__ void max_run(const unsigned long long* __restrict__ code, int64_t n, int shift,
                        unsigned long long* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long key = shift >= 64 ? 0ull : code[i] >> shift;
  if (i > 0) {
    unsigned long long prev = shift >= 64 ? 0ull : code[i - 1] >> shift;
    if (prev == key) return;
  }
  // upper bound of key in [i, n)
  int64_t lo = i, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    unsigned long long v = shift >= 64 ? 0ull : code[mid] >> shift;
    if (v <= key) lo = mid + 1;
    else hi = mid;
  }
  atomicMax(out, (unsigned long long)(lo - i));
}

__global__ void shift_codes(const unsigned long long* __restrict__ in, int64_t n, int shift,
                            unsigned long long* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] >> shift;
}

__global__ void iota64(int64_t* a, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

__global__ void gather_soa(const double* __restrict__ aos, const int64_t* __restrict__ perm, int64_t n, int d,
                           double* __restrict__ soa) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t src = perm[i];
  for (int k = 0; k < d; k++) soa[k * n + i] = aos[src * d + k];
}

// out[c] = lower_bound(sorted[0..n), keys[c]) ; out[nk] = n
__global__ void lower_bounds(const unsigned long long* __restrict__ sorted, int64_t n,
                             const unsigned long long* __restrict__ keys, int64_t nk, int64_t* __restrict__ out) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > nk) return;
  if (c == nk) {
    out[c] = n;
    return;
  }
  unsigned long long key = keys[c];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (sorted[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  out[c] = lo;
}

__global__ void gather_ptr(const int64_t* __restrict__ child_ptr, const int64_t* __restrict__ ch_ptr, int64_t n,
                           int64_t* __restrict__ out) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c <= n) out[c] = child_ptr[ch_ptr[c]];
}

// parent index of each cell of the finer level
__global__ void parent_of(const unsigned long long* __restrict__ child_code, int64_t nc, int D,
                          const unsigned long long* __restrict__ pcode, int64_t np_, int64_t* __restrict__ parent) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nc) return;
  unsigned long long key = child_code[c] >> D;
  int64_t lo = 0, hi = np_;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (pcode[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  parent[c] = lo;
}

template <int D>
__device__ __forceinline__ void deinterleave(unsigned long long code, int level, long long* mi) {
#pragma unroll
  for (int k = 0; k < D; k++) mi[k] = 0;
  for (int j = 0; j < level; j++) {
#pragma unroll
    for (int k = 0; k < D; k++) {
      int bitpos = (level - 1 - j) * D + (D - 1 - k);
      mi[k] = (mi[k] << 1) | (long long)((code >> bitpos) & 1ull);
    }
  }
}

template <int D>
__global__ void rm_keys(const unsigned long long* __restrict__ code, int64_t n, int level,
                        int64_t* __restrict__ rmkey) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  long long mi[D];
  deinterleave<D>(code[c], level, mi);
  long long k = 0;
#pragma unroll
  for (int q = 0; q < D; q++) k = (k << level) | mi[q];
  rmkey[c] = k;
}

__global__ void scatter_inv(const int64_t* __restrict__ perm, int64_t n, int64_t* __restrict__ inv) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) inv[perm[i]] = i;
}

struct AdmParams {
  double lo0[H2B_MAXD];
  double wl, hw, diam, eta;
};

// geometry.py:147 boxes_admissible with the reference's roundings
template <int D>
__device__ __forceinline__ bool admissible_cells(const long long* ma, const long long* mb, const AdmParams& ap) {
  double dot = 0.0;
  double hw2 = __dadd_rn(ap.hw, ap.hw);
#pragma unroll
  for (int k = 0; k < D; k++) {
    double ca = __dadd_rn(ap.lo0[k], __dmul_rn((double)ma[k] + 0.5, ap.wl));
    double cb = __dadd_rn(ap.lo0[k], __dmul_rn((double)mb[k] + 0.5, ap.wl));
    double g = __dsub_rn(fabs(__dsub_rn(ca, cb)), hw2);
    g = g > 0.0 ? g : 0.0;
    dot = __fma_rn(g, g, dot);
  }
  return ap.diam <= __dmul_rn(ap.eta, __dsqrt_rn(dot));
}

// pass 0: counts; pass 1: fill (member index + its row-major key)
template <int D>
__global__ void build_lists(int pass, int level, int64_t n, const unsigned long long* __restrict__ code,
                            const int64_t* __restrict__ parent, const int64_t* __restrict__ pnb_ptr,
                            const int64_t* __restrict__ pnb_idx, const int64_t* __restrict__ pch_ptr,
                            const int64_t* __restrict__ rmkey, AdmParams ap, int64_t* __restrict__ nb_cnt,
                            int64_t* __restrict__ il_cnt, const int64_t* __restrict__ nb_ptr,
                            const int64_t* __restrict__ il_ptr, int64_t* __restrict__ nb_idx,
                            int64_t* __restrict__ il_idx, int64_t* __restrict__ nb_key,
                            int64_t* __restrict__ il_key) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= n) return;
  long long mb[D], mc[D];
  deinterleave<D>(code[b], level, mb);
  int64_t p = parent[b];
  int64_t cn = 0, ci = 0, wn = 0, wi = 0;
  if (pass) {
    wn = nb_ptr[b];
    wi = il_ptr[b];
  }
  for (int64_t q = pnb_ptr[p]; q < pnb_ptr[p + 1]; q++) {
    int64_t nb = pnb_idx[q];
    for (int64_t c = pch_ptr[nb]; c < pch_ptr[nb + 1]; c++) {
      deinterleave<D>(code[c], level, mc);
      bool adm = admissible_cells<D>(mb, mc, ap);
      if (!pass) {
        if (adm) ci++;
        else cn++;
      } else if (adm) {
        il_idx[wi] = c;
        il_key[wi++] = rmkey[c];
      } else {
        nb_idx[wn] = c;
        nb_key[wn++] = rmkey[c];
      }
    }
  }
  if (!pass) {
    nb_cnt[b] = cn;
    il_cnt[b] = ci;
  }
}

// Sort every (short) list segment by its row-major key: one warp per segment,
// keys staged in shared memory, each element placed at its rank (keys within a
// segment are distinct cell keys).  Replaces a segmented radix sort whose
// launch overhead dominated for ~100-entry segments.
constexpr int SEG_SMAX = 512;  // longest segment handled here (longer -> CUB)
__global__ void rank_sort_segments(int64_t nseg, const int64_t* __restrict__ ptr, const int64_t* __restrict__ key,
                                   const int64_t* __restrict__ val, int64_t* __restrict__ out) {
  __shared__ int64_t ks[4][SEG_SMAX];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t seg = blockIdx.x * 4 + w;
  if (seg >= nseg) return;
  const int64_t b = ptr[seg], len = ptr[seg + 1] - b;
  for (int64_t i = lane; i < len; i += 32) ks[w][i] = key[b + i];
  __syncwarp();
  for (int64_t i = lane; i < len; i += 32) {
    const int64_t ki = ks[w][i];
    int r = 0;
    for (int64_t j = 0; j < len; j++) r += ks[w][j] < ki || (ks[w][j] == ki && j < i);
    out[b + r] = val[b + i];
  }
}

__global__ void max_seg_len(int64_t n, const int64_t* __restrict__ ptr, int* __restrict__ mx) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t len = ptr[c + 1] - ptr[c];
  atomicMax(mx, len > (1 << 30) ? (1 << 30) : (int)len);
}

struct Cub {
  DBuf<unsigned char> tmp;
  void ensure(size_t bytes) {
    if (tmp.n < bytes) tmp.alloc(bytes);
  }
};

void exclusive_scan_n1(const int64_t* cnt, int64_t n, int64_t* ptr, Cub& cub_, cudaStream_t s) {
  // ptr has n+1 entries; cnt has n entries (cnt may alias nothing)
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt, ptr, n + 1, s));
  cub_.ensure(bytes);
  CK(cub::DeviceScan::ExclusiveSum(cub_.tmp.get(), bytes, cnt, ptr, n + 1, s));
}

template <int D>
void build_tree_impl(DevTree& T, const double* Pd, const double* Qd, cudaStream_t s) {
  const int d = D;
  Cub cub_;
  const int64_t np = T.np, nq = T.nq;
  // ---------------- root box (geometry.py:243-247) ----------------
  {
    int nb = 512;
    DBuf<double> lo, hi;
    lo.alloc(nb * d);
    hi.alloc(nb * d);
    std::vector<double> l(d, INFINITY), h(d, -INFINITY);
    for (int pass = 0; pass < (T.shared ? 1 : 2); pass++) {
      const double* src = pass ? Qd : Pd;
      int64_t n = pass ? nq : np;
      bbox_partial<<<nb, 256, 0, s>>>(src, n, d, lo.get(), hi.get());
      CKL();
      auto hl = to_host(lo.get(), nb * d, s), hh = to_host(hi.get(), nb * d, s);
      for (int b = 0; b < nb; b++)
        for (int k = 0; k < d; k++) {
          l[k] = std::fmin(l[k], hl[b * d + k]);
          h[k] = std::fmax(h[k], hh[b * d + k]);
        }
    }
    double hm = -INFINITY;
    for (int k = 0; k < d; k++) {
      volatile double sum = l[k] + h[k];
      T.mid[k] = 0.5 * sum;
      volatile double e = h[k] - T.mid[k];
      if (e > hm) hm = e;
    }
    double half = hm > 0 ? hm : 1.0;
    half *= 1.0 + 1e-12;
    T.half = half;
    for (int k = 0; k < d; k++) T.lo0[k] = T.mid[k] - half;
  }
  // ---------------- Morton codes ----------------
  // deepest level the reference can address before np.ravel_multi_index
  // overflows (geometry.py:303) or the width underflow stop (geometry.py:269)
  int Lcap = std::min(50, 62 / d);
  T.Lmax = Lcap;
  BinParams bp;
  for (int k = 0; k < d; k++) bp.lo0[k] = T.lo0[k];
  for (int l = 0; l < Lcap; l++) bp.w2[l] = 2.0 * (T.half * std::ldexp(1.0, -l));
  const int nsets = T.shared ? 1 : 2;
  DBuf<unsigned long long> code_raw[2], code_sorted[2];
  DBuf<int64_t> idx_raw[2], idx_sorted[2];
  for (int set = 0; set < nsets; set++) {
    const double* src = set ? Qd : Pd;
    int64_t n = set ? nq : np;
    code_raw[set].alloc(n);
    code_sorted[set].alloc(n);
    idx_raw[set].alloc(n);
    idx_sorted[set].alloc(n);
    morton_codes<D><<<ceil_div(n, 256), 256, 0, s>>>(src, n, Lcap, bp, code_raw[set].get(), idx_raw[set].get());
    CKL();
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, code_raw[set].get(), code_sorted[set].get(),
                                       idx_raw[set].get(), idx_sorted[set].get(), n, 0, d * Lcap, s));
    cub_.ensure(bytes);
    CK(cub::DeviceRadixSort::SortPairs(cub_.tmp.get(), bytes, code_raw[set].get(), code_sorted[set].get(),
                                       idx_raw[set].get(), idx_sorted[set].get(), n, 0, d * Lcap, s));
  }
  // ---------------- depth (geometry.py:262-314 loop control) ----------------
  DBuf<unsigned long long> runbuf;
  runbuf.alloc(1);
  auto worst_at = [&](int level) -> int64_t {
    unsigned long long best = 0;
    for (int set = 0; set < nsets; set++) {
      int64_t n = set ? nq : np;
      CK(cudaMemsetAsync(runbuf.get(), 0, sizeof(unsigned long long), s));
      max_run<<<ceil_div(n, 256), 256, 0, s>>>(code_sorted[set].get(), n, d * (Lcap - level), runbuf.get());
      CKL();
      best = std::max(best, read_one(runbuf.get(), s));
    }
    return (int64_t)best;
  };
  int level = 0;
  int64_t worst = std::max(np, nq);
  for (;;) {
    if (worst <= T.nu) break;
    double width = T.half * std::ldexp(1.0, -level);
    if (width / (2.0 * T.half) < WIDTH_UNDERFLOW) {
      T.over_capacity = 1;
      break;
    }
    if ((int64_t)(level + 1) * d >= 63)
      throw std::invalid_argument(
          "invalid dims: array size defined by dims is larger than the maximum possible size.");
    level++;
    if (level > Lcap) throw std::runtime_error("tree deeper than the Morton code capacity");
    worst = worst_at(level);
  }
  const int L = level;
  T.depth = L;
  // ---------------- final point order: (leaf cell, index) ----------------
  const int shiftL = d * (Lcap - L);
  DBuf<unsigned long long> leaf_sorted[2];
  for (int set = 0; set < nsets; set++) {
    int64_t n = set ? nq : np;
    DBuf<unsigned long long> leaf_raw;
    leaf_raw.alloc(n);
    leaf_sorted[set].alloc(n);
    shift_codes<<<ceil_div(n, 256), 256, 0, s>>>(code_raw[set].get(), n, shiftL, leaf_raw.get());
    CKL();
    iota64<<<ceil_div(n, 256), 256, 0, s>>>(idx_raw[set].get(), n);
    CKL();
    DBuf<int64_t>& perm = set ? T.s_perm : T.t_perm;
    perm.alloc(n, &T.mem);
    size_t bytes = 0;
    int endbit = std::max(1, d * L);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, leaf_raw.get(), leaf_sorted[set].get(), idx_raw[set].get(),
                                       perm.get(), n, 0, endbit, s));
    cub_.ensure(bytes);
    CK(cub::DeviceRadixSort::SortPairs(cub_.tmp.get(), bytes, leaf_raw.get(), leaf_sorted[set].get(),
                                       idx_raw[set].get(), perm.get(), n, 0, endbit, s));
    DBuf<double>& soa = set ? T.ss : T.ts;
    soa.alloc(n * d, &T.mem);
    gather_soa<<<ceil_div(n, 256), 256, 0, s>>>(set ? Qd : Pd, perm.get(), n, d, soa.get());
    CKL();
    code_raw[set].release();
    code_sorted[set].release();
    idx_sorted[set].release();
  }
  // ---------------- cells per level ----------------
  T.lv.clear();
  T.lv.resize(L + 1);
  {
    // leaf cells = unique(leaf codes of targets U sources)
    DevLevel& LL = T.lv[L];
    int64_t ntot = np + (T.shared ? 0 : nq);
    DBuf<unsigned long long> all, uniq;
    DBuf<int64_t> nsel;
    all.alloc(ntot);
    uniq.alloc(ntot);
    nsel.alloc(1);
    CK(cudaMemcpyAsync(all.get(), leaf_sorted[0].get(), np * 8, cudaMemcpyDeviceToDevice, s));
    if (!T.shared) {
      CK(cudaMemcpyAsync(all.get() + np, leaf_sorted[1].get(), nq * 8, cudaMemcpyDeviceToDevice, s));
      DBuf<unsigned long long> srt;
      srt.alloc(ntot);
      size_t bytes = 0;
      int endbit = std::max(1, d * L);
      CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, all.get(), srt.get(), ntot, 0, endbit, s));
      cub_.ensure(bytes);
      CK(cub::DeviceRadixSort::SortKeys(cub_.tmp.get(), bytes, all.get(), srt.get(), ntot, 0, endbit, s));
      all = std::move(srt);
    }
    size_t bytes = 0;
    CK(cub::DeviceSelect::Unique(nullptr, bytes, all.get(), uniq.get(), nsel.get(), ntot, s));
    cub_.ensure(bytes);
    CK(cub::DeviceSelect::Unique(cub_.tmp.get(), bytes, all.get(), uniq.get(), nsel.get(), ntot, s));
    LL.n = read_one(nsel.get(), s);
    LL.code.alloc(LL.n, &T.mem);
    CK(cudaMemcpyAsync(LL.code.get(), uniq.get(), LL.n * 8, cudaMemcpyDeviceToDevice, s));
    LL.t_ptr.alloc(LL.n + 1, &T.mem);
    lower_bounds<<<ceil_div(LL.n + 1, 256), 256, 0, s>>>(leaf_sorted[0].get(), np, LL.code.get(), LL.n,
                                                         LL.t_ptr.get());
    CKL();
    if (!T.shared) {
      LL.s_ptr.alloc(LL.n + 1, &T.mem);
      lower_bounds<<<ceil_div(LL.n + 1, 256), 256, 0, s>>>(leaf_sorted[1].get(), nq, LL.code.get(), LL.n,
                                                           LL.s_ptr.get());
      CKL();
    }
    LL.ch_ptr.alloc(LL.n + 1, &T.mem);
    CK(cudaMemsetAsync(LL.ch_ptr.get(), 0, (LL.n + 1) * 8, s));
  }
  for (int l = L - 1; l >= 0; l--) {
    DevLevel& C = T.lv[l + 1];
    DevLevel& Pl = T.lv[l];
    DBuf<unsigned long long> pc, uniq;
    DBuf<int64_t> nsel;
    pc.alloc(C.n);
    uniq.alloc(C.n);
    nsel.alloc(1);
    shift_codes<<<ceil_div(C.n, 256), 256, 0, s>>>(C.code.get(), C.n, d, pc.get());
    CKL();
    size_t bytes = 0;
    CK(cub::DeviceSelect::Unique(nullptr, bytes, pc.get(), uniq.get(), nsel.get(), C.n, s));
    cub_.ensure(bytes);
    CK(cub::DeviceSelect::Unique(cub_.tmp.get(), bytes, pc.get(), uniq.get(), nsel.get(), C.n, s));
    Pl.n = read_one(nsel.get(), s);
    Pl.code.alloc(Pl.n, &T.mem);
    CK(cudaMemcpyAsync(Pl.code.get(), uniq.get(), Pl.n * 8, cudaMemcpyDeviceToDevice, s));
    C.parent.alloc(C.n, &T.mem);
    parent_of<<<ceil_div(C.n, 256), 256, 0, s>>>(C.code.get(), C.n, d, Pl.code.get(), Pl.n, C.parent.get());
    CKL();
    Pl.ch_ptr.alloc(Pl.n + 1, &T.mem);
    lower_bounds<<<ceil_div(Pl.n + 1, 256), 256, 0, s>>>(pc.get(), C.n, Pl.code.get(), Pl.n, Pl.ch_ptr.get());
    CKL();
    Pl.t_ptr.alloc(Pl.n + 1, &T.mem);
    gather_ptr<<<ceil_div(Pl.n + 1, 256), 256, 0, s>>>(C.t_ptr.get(), Pl.ch_ptr.get(), Pl.n, Pl.t_ptr.get());
    CKL();
    if (!T.shared) {
      Pl.s_ptr.alloc(Pl.n + 1, &T.mem);
      gather_ptr<<<ceil_div(Pl.n + 1, 256), 256, 0, s>>>(C.s_ptr.get(), Pl.ch_ptr.get(), Pl.n, Pl.s_ptr.get());
      CKL();
    }
  }
  T.lv[0].parent.alloc(1, &T.mem);
  CK(cudaMemsetAsync(T.lv[0].parent.get(), 0xff, 8, s));  // -1
  // ---------------- reference order (row-major keys) ----------------
  for (int l = 0; l <= L; l++) {
    DevLevel& V = T.lv[l];
    V.rmkey.alloc(V.n, &T.mem);
    rm_keys<D><<<ceil_div(V.n, 256), 256, 0, s>>>(V.code.get(), V.n, l, V.rmkey.get());
    CKL();
    DBuf<int64_t> keys_sorted, iota;
    keys_sorted.alloc(V.n);
    iota.alloc(V.n);
    iota64<<<ceil_div(V.n, 256), 256, 0, s>>>(iota.get(), V.n);
    CKL();
    V.rm_perm.alloc(V.n, &T.mem);
    V.rm_inv.alloc(V.n, &T.mem);
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, V.rmkey.get(), keys_sorted.get(), iota.get(),
                                       V.rm_perm.get(), V.n, 0, std::max(1, d * l), s));
    cub_.ensure(bytes);
    CK(cub::DeviceRadixSort::SortPairs(cub_.tmp.get(), bytes, V.rmkey.get(), keys_sorted.get(), iota.get(),
                                       V.rm_perm.get(), V.n, 0, std::max(1, d * l), s));
    scatter_inv<<<ceil_div(V.n, 256), 256, 0, s>>>(V.rm_perm.get(), V.n, V.rm_inv.get());
    CKL();
  }
  // ---------------- lists ----------------
  {
    DevLevel& R = T.lv[0];
    R.nb_ptr.alloc(2, &T.mem);
    R.nb_idx.alloc(1, &T.mem);
    R.il_ptr.alloc(2, &T.mem);
    R.il_idx.alloc(1, &T.mem);
    int64_t hp[2] = {0, 1}, zero[2] = {0, 0};
    CK(cudaMemcpyAsync(R.nb_ptr.get(), hp, 16, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(R.nb_idx.get(), zero, 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(R.il_ptr.get(), zero, 16, cudaMemcpyHostToDevice, s));
    R.nb_total = 1;
    R.il_total = 0;
    CK(cudaStreamSynchronize(s));
  }
  for (int l = 1; l <= L; l++) {
    DevLevel& V = T.lv[l];
    const DevLevel& Pl = T.lv[l - 1];
    AdmParams ap;
    for (int k = 0; k < d; k++) ap.lo0[k] = T.lo0[k];
    ap.wl = T.half * std::ldexp(1.0, 1 - l);
    ap.hw = 0.5 * ap.wl;
    ap.diam = 2.0 * ap.hw * std::sqrt((double)d);
    ap.eta = T.eta;
    DBuf<int64_t> nbc, ilc;
    nbc.alloc(V.n + 1);
    ilc.alloc(V.n + 1);
    CK(cudaMemsetAsync(nbc.get() + V.n, 0, 8, s));
    CK(cudaMemsetAsync(ilc.get() + V.n, 0, 8, s));
    unsigned g = ceil_div(V.n, 128);
    build_lists<D><<<g, 128, 0, s>>>(0, l, V.n, V.code.get(), V.parent.get(), Pl.nb_ptr.get(), Pl.nb_idx.get(),
                                     Pl.ch_ptr.get(), V.rmkey.get(), ap, nbc.get(), ilc.get(), nullptr, nullptr,
                                     nullptr, nullptr, nullptr, nullptr);
    CKL();
    V.nb_ptr.alloc(V.n + 1, &T.mem);
    V.il_ptr.alloc(V.n + 1, &T.mem);
    exclusive_scan_n1(nbc.get(), V.n, V.nb_ptr.get(), cub_, s);
    exclusive_scan_n1(ilc.get(), V.n, V.il_ptr.get(), cub_, s);
    V.nb_total = read_one(V.nb_ptr.get() + V.n, s);
    V.il_total = read_one(V.il_ptr.get() + V.n, s);
    DBuf<int64_t> nbk, ilk, nbi, ili;
    nbk.alloc(std::max<int64_t>(V.nb_total, 1));
    ilk.alloc(std::max<int64_t>(V.il_total, 1));
    nbi.alloc(std::max<int64_t>(V.nb_total, 1));
    ili.alloc(std::max<int64_t>(V.il_total, 1));
    build_lists<D><<<g, 128, 0, s>>>(1, l, V.n, V.code.get(), V.parent.get(), Pl.nb_ptr.get(), Pl.nb_idx.get(),
                                     Pl.ch_ptr.get(), V.rmkey.get(), ap, nullptr, nullptr, V.nb_ptr.get(),
                                     V.il_ptr.get(), nbi.get(), ili.get(), nbk.get(), ilk.get());
    CKL();
    V.nb_idx.alloc(std::max<int64_t>(V.nb_total, 1), &T.mem);
    V.il_idx.alloc(std::max<int64_t>(V.il_total, 1), &T.mem);
    for (int which = 0; which < 2; which++) {
      int64_t tot = which ? V.il_total : V.nb_total;
      if (!tot) continue;
      const int64_t* sp = which ? V.il_ptr.get() : V.nb_ptr.get();
      DBuf<int> mx;
      mx.alloc(1);
      CK(cudaMemsetAsync(mx.get(), 0, sizeof(int), s));
      max_seg_len<<<nblk(V.n, 256), 256, 0, s>>>(V.n, sp, mx.get());
      CKL();
      if (read_one(mx.get(), s) <= SEG_SMAX) {
        rank_sort_segments<<<ceil_div(V.n, 4), 128, 0, s>>>(V.n, sp, which ? ilk.get() : nbk.get(),
                                                             which ? ili.get() : nbi.get(),
                                                             which ? V.il_idx.get() : V.nb_idx.get());
        CKL();
        continue;
      }
      DBuf<int64_t> ksorted;
      ksorted.alloc(tot);
      const int64_t* ptr = which ? V.il_ptr.get() : V.nb_ptr.get();
      size_t bytes = 0;
      CK(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, which ? ilk.get() : nbk.get(), ksorted.get(),
                                             which ? ili.get() : nbi.get(), which ? V.il_idx.get() : V.nb_idx.get(),
                                             tot, V.n, ptr, ptr + 1, s));
      cub_.ensure(bytes);
      CK(cub::DeviceSegmentedSort::SortPairs(cub_.tmp.get(), bytes, which ? ilk.get() : nbk.get(), ksorted.get(),
                                             which ? ili.get() : nbi.get(), which ? V.il_idx.get() : V.nb_idx.get(),
                                             tot, V.n, ptr, ptr + 1, s));
    }
    CK(cudaStreamSynchronize(s));
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace

std::unique_ptr<DevTree> build_tree(const double* P, int64_t np, const double* Q, int64_t nq, int d, int shared,
                                    int64_t nu, double eta, bool on_device, cudaStream_t s) {
  // geometry.py:235-240 argument checks
  if (np == 0 || nq == 0) throw std::invalid_argument("empty point set");
  if (nu < 1) throw std::invalid_argument("invalid leaf capacity");
  if (!(eta > 0)) throw std::invalid_argument("eta must be positive");
  if (d < 1 || d > H2B_MAXD) throw std::invalid_argument("dimension must be between 1 and 4");
  if (shared && np != nq) throw std::invalid_argument("shared cloud needs equal point counts");
  auto T = std::make_unique<DevTree>();
  T->d = d;
  T->np = np;
  T->nq = nq;
  T->nu = nu;
  T->eta = eta;
  T->shared = shared;
  T->P.alloc(np * d, &T->mem);
  CK(cudaMemcpyAsync(T->P.get(), P, np * d * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  if (!shared) {
    T->Q.alloc(nq * d, &T->mem);
    CK(cudaMemcpyAsync(T->Q.get(), Q, nq * d * 8, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       s));
  }
  switch (d) {
    case 1: build_tree_impl<1>(*T, T->Pd(), T->Qd(), s); break;
    case 2: build_tree_impl<2>(*T, T->Pd(), T->Qd(), s); break;
    case 3: build_tree_impl<3>(*T, T->Pd(), T->Qd(), s); break;
    default: build_tree_impl<4>(*T, T->Pd(), T->Qd(), s); break;
  }
  return T;
}

}  // namespace h2b
