// common.cuh — shared device helpers for the B200 NNCA / H2 engine.
//
// Two families of kernel evaluators:
//   * kval_exact / r2_exact: the reference's arithmetic (_core.pyx:15 _kval,
//     :38 _r2) with every rounding pinned by __d*_rn intrinsics so nvcc
//     cannot contract into FMAs.  Used wherever results feed a discrete
//     decision (ACA pivot search) or are compared bit-for-bit.
//   * the fast evaluators in interact.cuh: FMA-contracted distance, MUFU
//     rsqrt + Newton, used in the matvec (tolerance 1e-10 relative).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#define H2B_MAXD 4

namespace h2b {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw ::h2b::cuda_error(std::string(#x) + ": " + cudaGetErrorString(e_) + " @" __FILE__ \
                              ":" + std::to_string(__LINE__));                                 \
  } while (0)

#define CKL() CK(cudaGetLastError())

constexpr double INV_FOUR_PI = 0.07957747154594767;

enum Kind {
  REG_LOG = 0,
  REG_INVERSE = 1,
  COULOMB = 2,
  MATERN = 3,
  GAUSSIAN = 4,
  LAPLACE = 5,
  LOG = 6,
  GAUSSIAN_SCALED = 7
};

__host__ __device__ inline bool kind_valid(int k) { return k >= 0 && k <= 7; }

// ---------------------------------------------------------------------
// exact (reference-rounding) evaluation
// ---------------------------------------------------------------------
__device__ __forceinline__ double kval_exact(int kind, double a, double r2) {
  if (kind == GAUSSIAN) return exp(-r2);
  if (kind == GAUSSIAN_SCALED) return exp(-__dmul_rn(a, r2));
  double r = __dsqrt_rn(r2);
  switch (kind) {
    case MATERN:
      return exp(-r);
    case COULOMB:
      return r == 0.0 ? 0.0 : __ddiv_rn(1.0, r);
    case LAPLACE:
      return r == 0.0 ? 0.0 : __ddiv_rn(INV_FOUR_PI, r);
    case LOG:
      return r == 0.0 ? 0.0 : log(r);
    case REG_INVERSE:
      return r < a ? __ddiv_rn(r, a) : __ddiv_rn(a, r);
    default:  // REG_LOG
      if (r >= a) return __ddiv_rn(log(r), log(a));
      if (r == 0.0) return 0.0;
      return __ddiv_rn(__dmul_rn(r, __dsub_rn(log(r), 1.0)), __dmul_rn(a, __dsub_rn(log(a), 1.0)));
  }
}

// sum_k (x_k - y_k)^2 accumulated left to right from 0.0, no FMA (_core.pyx:38)
template <int D>
__device__ __forceinline__ double r2_exact(const double* x, const double* y) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < D; k++) {
    double df = __dsub_rn(x[k], y[k]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  return acc;
}

// ---------------------------------------------------------------------
// warp / block reductions
// ---------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// argmax with ties to the lowest index; idx < 0 marks "none"
__device__ __forceinline__ void argmax_merge(double& v, int64_t& i, double v2, int64_t i2) {
  if (i2 < 0) return;
  if (i < 0 || v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__device__ __forceinline__ void warp_argmax(double& v, int64_t& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    long long i2 = __shfl_xor_sync(0xffffffffu, (long long)i, o);
    argmax_merge(v, i, v2, i2);
  }
}

// The same for values >= 0 (|residual| candidates) and indices < 2^31, with warp-wide integer reductions
// (REDUX): the bit pattern of a non-negative double orders like an unsigned integer, so the maximum is the
// maximum high word, then the maximum low word among its holders, then the lowest index among those.  Three
// REDUX instead of five rounds of four shuffles + merge logic; the pivot search runs twice per ACA step.
__device__ __forceinline__ void warp_argmax_nn(double& v, int64_t& i) {
  const bool has = i >= 0;
  const unsigned hi = has ? (unsigned)__double2hiint(v) : 0u;
  const unsigned lo = has ? (unsigned)__double2loint(v) : 0u;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const bool c1 = has && hi == mh;
  const unsigned ml = __reduce_max_sync(0xffffffffu, c1 ? lo : 0u);
  const bool c2 = c1 && lo == ml;
  const unsigned mi = __reduce_min_sync(0xffffffffu, c2 ? (unsigned)i : 0xffffffffu);
  if (mi == 0xffffffffu) {
    v = -1.0;
    i = -1;
  } else {
    v = __hiloint2double((int)mh, (int)ml);
    i = (int64_t)mi;
  }
}

__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long v2 = __shfl_xor_sync(0xffffffffu, (long long)v, o);
    v = v2 < v ? v2 : v;
  }
  return v;
}

// ---- mbarrier / TMA bulk-copy helpers (sm_90+ PTX, used on sm_100a) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the same with precomputed shared-memory addresses (hot loops)
__device__ __forceinline__ void mbar_expect_tx_u32(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
  // with a suspend-time hint the warp sleeps in hardware between polls instead of spinning through the loop
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 0x989680;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// generic-proxy smem writes (the in-place transform) before a later TMA write
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// generic-proxy global writes (residual rows) before a later TMA read of them
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// ---------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------
inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }
// grid size for a bounds-checked 1D kernel: never 0 (a 0-block launch is an error)
inline unsigned nblk(int64_t n, int64_t b) { return n > 0 ? ceil_div(n, b) : 1u; }

// Stream-ordered allocation: every DBuf is carved from the device's default
// memory pool (cudaMallocAsync) on the stream of the current API call, and
// the pool keeps freed memory cached (release threshold = max), so the many
// short-lived workspaces of the setup cost no cudaMalloc/cudaFree round trips.
inline cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = 0;
  return s;
}
struct StreamScope {
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~StreamScope() { alloc_stream() = prev; }
};
inline void pool_init() {
  // once per device (a process may drive several GPUs)
  static std::once_flag flags[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::call_once(flags[dev & 63], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      // Up-front reservation: later allocations are carved from already-mapped
      // memory.  Without it, pool growth in the middle of a setup (mapping
      // new physical pages) made random setups 2-3x slower (measured: NNCA
      // 195 ms steady vs 210-700 ms).  Default min(24 GB, 20% of the device);
      // H2B_POOL_RESERVE_GB overrides (0 disables).
      const char* e = getenv("H2B_POOL_RESERVE_GB");
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      size_t bytes = e ? ((size_t)atol(e) << 30) : std::min<size_t>((size_t)24 << 30, tot / 5);
      bytes = std::min(bytes, fr / 2);
      const size_t gb = bytes >> 30;
      if (gb) {
        void* p = nullptr;
        if (cudaMallocAsync(&p, gb << 30, 0) == cudaSuccess) cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
      }
    }
  });
}

// Device buffer with byte accounting.
struct MemStats {
  int64_t bytes = 0;
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  MemStats* ms = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), ms(o.ms) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; ms = o.ms;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, MemStats* stats = nullptr) {
    release();
    n = count;
    ms = stats;
    if (count) {
      pool_init();
      CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), alloc_stream()));
      if (ms) ms->bytes += (int64_t)(count * sizeof(T));
    }
  }
  void release() {
    if (p) {
      cudaFreeAsync(p, alloc_stream());
      if (ms) ms->bytes -= (int64_t)(n * sizeof(T));
    }
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

template <class T>
inline std::vector<T> to_host(const T* d, size_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) {
    CK(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return h;
}

template <class T>
inline T read_one(const T* d, cudaStream_t s) {
  T v;
  CK(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return v;
}

}  // namespace h2b
