// capi.cu — extern "C" boundary of libh2b200.so (declared in include/h2b.h).
// Converts exceptions to return codes and maps the engine's Morton cell order
// to the reference's cell order (nonempty cells sorted by multi-index).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/h2b.h"
#include "engine.cuh"

namespace h2b {
void dense_rows_dev(int kind, double a, const double* P, const int64_t* rows, int64_t nrows, const double* Q,
                    int64_t nq, int d, const double* w, double* u, cudaStream_t s);
}

using namespace h2b;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("ValueError: ") + e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

struct LevelHost {
  bool ready = false;
  std::vector<int64_t> key, mi, t_ptr, t_idx, s_ptr, s_idx, nb_ptr, nb_idx, il_ptr, il_idx, parent, ch_ptr, ch_idx;
};

}  // namespace

// Stream discipline.  Every handle carries an event recorded after the last work submitted on its behalf.  A
// call on a different stream first makes that stream wait for the event (the per-H2 matvec scratch and the
// tree arrays are then never touched by two streams at once), host callers are serialised by the handle's
// mutex, and the free functions wait for the event before releasing device memory, so dropping a handle while
// its last product is still running on a non-blocking stream is safe.
struct Tail {
  cudaEvent_t ev = nullptr;
  cudaStream_t last = nullptr;
  bool used = false;
  void enter(cudaStream_t s) {  // order s after the previous call if that ran on another stream
    if (used && s != last && ev) CK(cudaStreamWaitEvent(s, ev, 0));
  }
  void leave(cudaStream_t s) {
    if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, s));
    last = s;
    used = true;
  }
  void drain() {  // host-side wait for the last submitted work, then drop the event
    if (ev) {
      cudaEventSynchronize(ev);
      cudaEventDestroy(ev);
      ev = nullptr;
    }
  }
};

struct h2b_tree {
  std::unique_ptr<DevTree> t;
  std::vector<LevelHost> host;
  std::vector<std::vector<int64_t>> perm, inv;  // per level (host copies)
  std::mutex mu;
  Tail tail;
};

struct h2b_h2 {
  std::unique_ptr<DevH2> h;
  h2b_tree* tree;
  std::mutex mu;
  Tail tail;
};

namespace {

void ensure_perm(h2b_tree* T, int level) {
  if ((int)T->perm.size() != T->t->depth + 1) {
    T->perm.assign(T->t->depth + 1, {});
    T->inv.assign(T->t->depth + 1, {});
    T->host.assign(T->t->depth + 1, LevelHost{});
  }
  if (T->perm[level].empty() && T->t->lv[level].n) {
    const DevLevel& L = T->t->lv[level];
    T->perm[level] = to_host(L.rm_perm.get(), L.n, 0);
    T->inv[level] = to_host(L.rm_inv.get(), L.n, 0);
  }
}

void ensure_host_level(h2b_tree* T, int level) {
  std::lock_guard<std::mutex> g(T->mu);
  ensure_perm(T, level);
  LevelHost& H = T->host[level];
  if (H.ready) return;
  const DevTree& t = *T->t;
  const DevLevel& L = t.lv[level];
  const int64_t n = L.n;
  const int d = t.d;
  auto& perm = T->perm[level];
  auto& inv = T->inv[level];
  auto rmkey = to_host(L.rmkey.get(), n, 0);
  auto tptr = to_host(L.t_ptr.get(), n + 1, 0);
  auto sptr = t.shared ? tptr : to_host(L.s_ptr.get(), n + 1, 0);
  auto tperm = to_host(t.t_perm.get(), t.np, 0);
  auto sperm = t.shared ? tperm : to_host(t.s_perm.get(), t.nq, 0);
  H.key.resize(n);
  H.mi.resize(n * d);
  for (int64_t i = 0; i < n; i++) {
    int64_t k = rmkey[perm[i]];
    H.key[i] = k;
    for (int q = d - 1; q >= 0; q--) {
      H.mi[i * d + q] = level ? (k & ((1LL << level) - 1)) : 0;
      k = level ? (k >> level) : 0;
    }
  }
  auto ranges = [&](const std::vector<int64_t>& ptr, const std::vector<int64_t>& pm, std::vector<int64_t>& optr,
                    std::vector<int64_t>& oidx) {
    optr.assign(n + 1, 0);
    for (int64_t i = 0; i < n; i++) optr[i + 1] = optr[i] + (ptr[perm[i] + 1] - ptr[perm[i]]);
    oidx.resize(optr[n]);
    for (int64_t i = 0; i < n; i++) {
      int64_t c = perm[i];
      std::copy(pm.begin() + ptr[c], pm.begin() + ptr[c + 1], oidx.begin() + optr[i]);
      std::sort(oidx.begin() + optr[i], oidx.begin() + optr[i + 1]);  // geometry.py:226 np.sort
    }
  };
  ranges(tptr, tperm, H.t_ptr, H.t_idx);
  ranges(sptr, sperm, H.s_ptr, H.s_idx);
  auto lists = [&](const DBuf<int64_t>& dptr, const DBuf<int64_t>& didx, int64_t tot, std::vector<int64_t>& optr,
                   std::vector<int64_t>& oidx) {
    auto ptr = to_host(dptr.get(), n + 1, 0);
    auto idx = to_host(didx.get(), std::max<int64_t>(tot, 0), 0);
    optr.assign(n + 1, 0);
    for (int64_t i = 0; i < n; i++) optr[i + 1] = optr[i] + (ptr[perm[i] + 1] - ptr[perm[i]]);
    oidx.resize(optr[n]);
    for (int64_t i = 0; i < n; i++) {
      int64_t c = perm[i], w = optr[i];
      for (int64_t q = ptr[c]; q < ptr[c + 1]; q++) oidx[w++] = inv[idx[q]];
    }
  };
  lists(L.nb_ptr, L.nb_idx, L.nb_total, H.nb_ptr, H.nb_idx);
  lists(L.il_ptr, L.il_idx, L.il_total, H.il_ptr, H.il_idx);
  H.parent.assign(n, -1);
  if (level > 0) {
    ensure_perm(T, level - 1);
    auto par = to_host(L.parent.get(), n, 0);
    for (int64_t i = 0; i < n; i++) H.parent[i] = T->inv[level - 1][par[perm[i]]];
  }
  H.ch_ptr.assign(n + 1, 0);
  H.ch_idx.clear();
  if (level < t.depth) {
    ensure_perm(T, level + 1);
    auto chp = to_host(L.ch_ptr.get(), n + 1, 0);
    for (int64_t i = 0; i < n; i++) {
      int64_t c = perm[i];
      for (int64_t q = chp[c]; q < chp[c + 1]; q++) H.ch_idx.push_back(T->inv[level + 1][q]);
      H.ch_ptr[i + 1] = (int64_t)H.ch_idx.size();
    }
  }
  H.ready = true;
}

}  // namespace

extern "C" {

const char* h2b_last_error(void) { return g_err.c_str(); }
int h2b_version(void) { return 1; }

int h2b_kernel_block(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d,
                     double* out) {
  return guarded([&] {
    if (!kind_valid(kind)) throw std::invalid_argument("unknown kernel kind");
    if (m * n == 0) return;
    DBuf<double> dx, dy, dout;
    dx.alloc(m * d);
    dy.alloc(n * d);
    dout.alloc(m * n);
    CK(cudaMemcpy(dx.get(), X, m * d * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dy.get(), Y, n * d * 8, cudaMemcpyHostToDevice));
    kernel_block(kind, a, dx.get(), m, dy.get(), n, d, dout.get(), 0);
    CK(cudaMemcpy(out, dout.get(), m * n * 8, cudaMemcpyDeviceToHost));
  });
}

int h2b_kernel_row(int kind, double a, const double* x, const double* Y, int64_t n, int d, double* out) {
  return h2b_kernel_block(kind, a, x, 1, Y, n, d, out);
}

int h2b_aca_kernel(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d, double eps,
                   int64_t cap, double* U, double* V, int64_t* rp, int64_t* cp, int* converged, int64_t* nevals,
                   int64_t* rank) {
  return guarded([&] {
    if (!kind_valid(kind)) throw std::invalid_argument("unknown kernel kind");
    if (!(eps > 0)) throw std::invalid_argument("epsilon must be positive");
    if (d < 1 || d > H2B_MAXD) throw std::invalid_argument("dimension must be between 1 and 4");
    aca_single(kind, a, X, m, Y, n, d, eps, cap, U, V, rp, cp, converged, nevals, rank);
  });
}

int h2b_tree_build(const double* P, int64_t np, const double* Q, int64_t nq, int d, int shared, int64_t nu,
                   double eta, int on_device, void* stream, h2b_tree** out) {
  return guarded([&] {
    auto T = new h2b_tree();
    try {
      StreamScope sc((cudaStream_t)stream);
      T->t = build_tree(P, np, Q, nq, d, shared, nu, eta, on_device != 0, (cudaStream_t)stream);
      T->tail.leave((cudaStream_t)stream);
    } catch (...) {
      delete T;
      throw;
    }
    *out = T;
  });
}

void h2b_tree_free(h2b_tree* t) {
  if (!t) return;
  t->tail.drain();  // free the H2 matrices built on a tree before the tree itself
  delete t;
}

int h2b_tree_info(const h2b_tree* t, int* depth, int* over_capacity, double* mid, double* half) {
  return guarded([&] {
    *depth = t->t->depth;
    *over_capacity = t->t->over_capacity;
    for (int k = 0; k < t->t->d; k++) mid[k] = t->t->mid[k];
    *half = t->t->half;
  });
}

int64_t h2b_tree_ncells(const h2b_tree* t, int level) {
  if (level < 0 || level > t->t->depth) return -1;
  return t->t->lv[level].n;
}

int64_t h2b_tree_get(const h2b_tree* tc, int level, int what, int64_t* dst) {
  h2b_tree* t = const_cast<h2b_tree*>(tc);
  int64_t ret = -1;
  int rc = guarded([&] {
    if (level < 0 || level > t->t->depth) throw std::invalid_argument("level out of range");
    ensure_host_level(t, level);
    LevelHost& H = t->host[level];
    const std::vector<int64_t>* v = nullptr;
    switch (what) {
      case 0: v = &H.key; break;
      case 1: v = &H.mi; break;
      case 2: v = &H.t_ptr; break;
      case 3: v = &H.t_idx; break;
      case 4: v = &H.s_ptr; break;
      case 5: v = &H.s_idx; break;
      case 6: v = &H.nb_ptr; break;
      case 7: v = &H.nb_idx; break;
      case 8: v = &H.il_ptr; break;
      case 9: v = &H.il_idx; break;
      case 10: v = &H.parent; break;
      case 11: v = &H.ch_ptr; break;
      case 12: v = &H.ch_idx; break;
      default: throw std::invalid_argument("bad field");
    }
    if (dst && !v->empty()) std::memcpy(dst, v->data(), v->size() * 8);
    ret = (int64_t)v->size();
  });
  return rc ? rc : ret;
}

int h2b_assemble(const h2b_tree* t, int kind, double a, double eps, int force_general, int64_t max_rank,
                 void* stream, h2b_h2** out) {
  return guarded([&] {
    auto H = new h2b_h2();
    H->tree = const_cast<h2b_tree*>(t);
    try {
      const cudaStream_t s = (cudaStream_t)stream;
      StreamScope sc(s);
      {
        std::lock_guard<std::mutex> g(H->tree->mu);
        H->tree->tail.enter(s);
      }
      H->h = assemble(*t->t, kind, a, eps, force_general != 0, max_rank, s);
      H->tail.leave(s);
      std::lock_guard<std::mutex> g(H->tree->mu);
      H->tree->tail.leave(s);
    } catch (...) {
      delete H;
      throw;
    }
    *out = H;
  });
}

void h2b_h2_free(h2b_h2* h) {
  if (!h) return;
  h->tail.drain();
  delete h;
}

int h2b_release_workspace(void) {
  return guarded([&] { release_workspace(); });
}

int64_t h2b_h2_get_i64(const h2b_h2* hc, int level, int what, int64_t* dst) {
  int64_t ret = 0;
  int rc = guarded([&] {
    const DevH2& h = *hc->h;
    if (level < 2 || level > h.t->depth) {
      ret = 0;
      return;
    }
    h2b_tree* T = hc->tree;
    {
      std::lock_guard<std::mutex> g(T->mu);
      ensure_perm(T, level);
    }
    const auto& perm = T->perm[level];
    const DevH2Level& L = h.lv[level];
    const int64_t n = L.n;
    auto per_cell = [&](const int64_t* dv) {
      auto v = to_host(dv, n, 0);
      std::vector<int64_t> o(n);
      for (int64_t i = 0; i < n; i++) o[i] = v[perm[i]];
      return o;
    };
    std::vector<int64_t> outv;
    if (what == 0) outv = per_cell(L.kin.get());
    else if (what == 1) outv = per_cell(L.koutd());
    else if (what == 6) outv = per_cell(L.nevals.get());
    else if (what == 7) outv = per_cell(L.conv.get());
    else if (what == 8) outv = per_cell(L.m_in.get());
    else if (what == 9) outv = per_cell(L.n_outd());
    else if (what >= 2 && what <= 5) {
      bool in_side = (what == 2 || what == 3);
      const int64_t* dptr = in_side ? L.in_ptr.get() : L.out_ptrd();
      int64_t tot = in_side ? L.in_total : L.out_total;
      const int64_t* didx;
      if (what == 2) didx = L.t_in.get();
      else if (what == 3) didx = L.s_in.get();
      else if (what == 4) didx = L.t_out.n ? L.t_out.get() : L.s_in.get();
      else didx = L.s_out.n ? L.s_out.get() : L.t_in.get();
      auto ptr = to_host(dptr, n + 1, 0);
      auto idx = to_host(didx, tot, 0);
      outv.reserve(tot);
      for (int64_t i = 0; i < n; i++) {
        int64_t c = perm[i];
        outv.insert(outv.end(), idx.begin() + ptr[c], idx.begin() + ptr[c + 1]);
      }
    } else
      throw std::invalid_argument("bad field");
    if (dst && !outv.empty()) std::memcpy(dst, outv.data(), outv.size() * 8);
    ret = (int64_t)outv.size();
  });
  return rc ? rc : ret;
}

int64_t h2b_h2_get_interp(const h2b_h2* hc, int level, int64_t cell, int which, int64_t* cols, double* dst) {
  int64_t ret = 0;
  int rc = guarded([&] {
    const DevH2& h = *hc->h;
    if (level < 2 || level > h.t->depth) throw std::invalid_argument("level out of range");
    h2b_tree* T = hc->tree;
    {
      std::lock_guard<std::mutex> g(T->mu);
      ensure_perm(T, level);
    }
    const DevH2Level& L = h.lv[level];
    if (cell < 0 || cell >= L.n) throw std::invalid_argument("cell out of range");
    int64_t c = T->perm[level][cell];
    int64_t rows = read_one((which == 0 ? L.m_in.get() : L.n_outd()) + c, 0);
    int64_t k = read_one((which == 0 ? L.kin.get() : L.koutd()) + c, 0);
    int64_t off = read_one((which == 0 ? L.pm_off.get() : L.qm_offd()) + c, 0);
    if (cols) *cols = k;
    if (dst && rows * k > 0) {
      auto v = to_host((which == 0 ? L.pmat.get() : L.qmatd()) + off, rows * k, 0);
      for (int64_t i = 0; i < rows; i++)
        for (int64_t s = 0; s < k; s++) dst[i * k + s] = v[s * rows + i];
    }
    ret = rows;
  });
  return rc ? rc : ret;
}

int64_t h2b_h2_get_coeffs(h2b_h2* hc, int level, int which, double* dst) {
  int64_t ret = 0;
  int rc = guarded([&] {
    std::lock_guard<std::mutex> g(hc->mu);
    DevH2& h = *hc->h;
    if (which != 0 && which != 1) throw std::invalid_argument("bad field");
    if (level < 2 || level > h.t->depth) {
      ret = 0;
      return;
    }
    if (h.last_nrhs != 1 || h.scratch_nrhs != 1)
      throw std::invalid_argument("the last product on this matrix was not a single-vector product");
    if (hc->tail.ev) CK(cudaEventSynchronize(hc->tail.ev));
    h2b_tree* T = hc->tree;
    {
      std::lock_guard<std::mutex> gt(T->mu);
      ensure_perm(T, level);
    }
    const auto& perm = T->perm[level];
    const DevH2Level& L = h.lv[level];
    const int64_t tot = which == 0 ? L.out_total : L.in_total;
    auto ptr = to_host(which == 0 ? L.out_ptrd() : L.in_ptr.get(), L.n + 1, 0);
    auto val = to_host((which == 0 ? h.wout[level] : h.uin[level]).get(), tot, 0);
    if (dst) {
      int64_t w = 0;
      for (int64_t i = 0; i < L.n; i++) {
        const int64_t c = perm[i];
        for (int64_t q = ptr[c]; q < ptr[c + 1]; q++) dst[w++] = val[q];
      }
    }
    ret = tot;
  });
  return rc ? rc : ret;
}

int h2b_h2_stats(const h2b_h2* hc, int64_t* st) {
  return guarded([&] {
    const DevH2& h = *hc->h;
    st[0] = h.evals_pivots;
    st[1] = h.evals_couplings;
    st[2] = h.evals_nearfield;
    st[3] = h.max_rank;
    st[4] = h.cells_visited;
    st[5] = h.mem.bytes;
    st[6] = h.symmetric;
    st[7] = h.setup_ns;
    st[8] = h.t->depth;
    st[9] = h.unconverged;
  });
}

int h2b_matvec(h2b_h2* hc, const double* w, double* u, int64_t nrhs, int on_device, void* stream) {
  return guarded([&] {
    DevH2& h = *hc->h;
    const DevTree& T = *h.t;
    if (nrhs < 1) throw std::invalid_argument("nrhs must be positive");
    cudaStream_t s = (cudaStream_t)stream;
    StreamScope sc(s);
    // the product writes per-H2 scratch: one caller at a time, and a new stream waits for the previous one
    std::lock_guard<std::mutex> g(hc->mu);
    hc->tail.enter(s);
    if (on_device) {
      matvec(h, w, u, nrhs, s);
      hc->tail.leave(s);
      return;
    }
    if ((int64_t)h.io_w.n < T.nq * nrhs) h.io_w.alloc(T.nq * nrhs);
    if ((int64_t)h.io_u.n < T.np * nrhs) h.io_u.alloc(T.np * nrhs);
    CK(cudaMemcpyAsync(h.io_w.get(), w, T.nq * nrhs * 8, cudaMemcpyHostToDevice, s));
    matvec(h, h.io_w.get(), h.io_u.get(), nrhs, s);
    CK(cudaMemcpyAsync(u, h.io_u.get(), T.np * nrhs * 8, cudaMemcpyDeviceToHost, s));
    hc->tail.leave(s);
    CK(cudaStreamSynchronize(s));
  });
}

/* page-locked host buffers for the host-pointer calls (copies from pinned memory run at the full PCIe rate) */
int h2b_host_alloc(void** p, int64_t bytes) {
  return guarded([&] {
    if (bytes < 0) throw std::invalid_argument("negative size");
    CK(cudaHostAlloc(p, (size_t)std::max<int64_t>(bytes, 1), cudaHostAllocDefault));
  });
}
void h2b_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int64_t h2b_matvec_launches(const h2b_h2* h, int64_t nrhs) { return matvec_launches(*h->h, nrhs); }

int h2b_set_profiling(int on) {
  set_profiling(on != 0);
  return 0;
}

int h2b_fp64_peak(double* tflops) {
  return guarded([&] { *tflops = fp64_peak_tflops(0); });
}

int h2b_last_stage_ms(double* ms5) {
  last_stage_ms(ms5);
  return 0;
}

int h2b_dense_matvec(int kind, double a, const double* P, int64_t np, const double* Q, int64_t nq, int d,
                     const double* w, double* u, int64_t nrhs, int on_device, void* stream) {
  return guarded([&] {
    if (!kind_valid(kind)) throw std::invalid_argument("unknown kernel kind");
    cudaStream_t s = (cudaStream_t)stream;
    StreamScope sc(s);
    if (on_device) {
      dense_matvec(kind, a, P, np, Q, nq, d, w, u, nrhs, s);
      return;
    }
    DBuf<double> dp, dq, dw, du;
    dp.alloc(np * d);
    dq.alloc(nq * d);
    dw.alloc(nq * nrhs);
    du.alloc(np * nrhs);
    CK(cudaMemcpyAsync(dp.get(), P, np * d * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dq.get(), Q, nq * d * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dw.get(), w, nq * nrhs * 8, cudaMemcpyHostToDevice, s));
    dense_matvec(kind, a, dp.get(), np, dq.get(), nq, d, dw.get(), du.get(), nrhs, s);
    CK(cudaMemcpyAsync(u, du.get(), np * nrhs * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

int h2b_dense_rows(int kind, double a, const double* P, int64_t np, const int64_t* rows, int64_t nrows,
                   const double* Q, int64_t nq, int d, const double* w, double* u) {
  return guarded([&] {
    if (!kind_valid(kind)) throw std::invalid_argument("unknown kernel kind");
    if (nrows == 0) return;
    for (int64_t i = 0; i < nrows; i++)
      if (rows[i] < 0 || rows[i] >= np) throw std::invalid_argument("row index out of range");
    DBuf<double> dp, dq, dw, du;
    DBuf<int64_t> dr;
    dp.alloc(np * d);
    dq.alloc(nq * d);
    dw.alloc(nq);
    du.alloc(nrows);
    dr.alloc(nrows);
    CK(cudaMemcpy(dp.get(), P, np * d * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dq.get(), Q, nq * d * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dw.get(), w, nq * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dr.get(), rows, nrows * 8, cudaMemcpyHostToDevice));
    dense_rows_dev(kind, a, dp.get(), dr.get(), nrows, dq.get(), nq, d, dw.get(), du.get(), 0);
    CK(cudaMemcpy(u, du.get(), nrows * 8, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
