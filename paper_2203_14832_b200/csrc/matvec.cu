// matvec.cu — level-batched H2 matrix-vector product (matvec.py:142 h2_matvec,
// the five passes of matvec.py:169 h2_matvec_reference), FP64 throughout.
//
// The coupling blocks S_{X,Y} = K(t_in^X, s_out^Y) and the near-field blocks
// are NOT stored (the reference stores both): both are regenerated in
// registers inside one interaction kernel, because on B200 evaluating 1/r in
// FP64 (~12 FP64 instructions / entry) is ~3x cheaper than streaming the
// stored 8-byte entry from HBM.  Transfer operators (P2M/M2M/L2L/L2P) are
// applied from compact copies without their identity rows (transfer.cuh) as
// batched small GEMVs; the Morton cell order keeps every operand contiguous.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "interact_sym.cuh"
#include "transfer.cuh"

namespace h2b {

namespace {

bool g_profile = false;
double g_stage_ms[5] = {0, 0, 0, 0, 0};

__global__ void gather_rows(const double* __restrict__ w, const int64_t* __restrict__ perm, int64_t n, int64_t R,
                            double* __restrict__ out, double* __restrict__ recq, int rs, double* __restrict__ zero) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n * R) return;
  int64_t p = i / R, r = i - p * R;
  const double v = w[perm[p] * R + r];
  out[i] = v;
  if (recq) recq[i * rs] = v;  // one RHS: also the charge slot of the source record (no separate pack pass)
  if (zero) zero[i] = 0.0;     // symmetric one-RHS product: clears the near-field accumulator (np == nq there)
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

void interact_sym_all(int d, int kind, const DevH2& h, int64_t R, int64_t r0, const KParams& kp, cudaStream_t s) {
  switch (d) {
    case 1: interact_sym_d<1>(kind, h, R, r0, kp, s); break;
    case 2: interact_sym_d<2>(kind, h, R, r0, kp, s); break;
    case 3: interact_sym_d<3>(kind, h, R, r0, kp, s); break;
    default: interact_sym_d<4>(kind, h, R, r0, kp, s); break;
  }
}

void pack_coords(int d, const DevH2& h, int nr, cudaStream_t s) {
  switch (d) {
    case 1: pack_coords_dim<1>(h, nr, s); break;
    case 2: pack_coords_dim<2>(h, nr, s); break;
    case 3: pack_coords_dim<3>(h, nr, s); break;
    default: pack_coords_dim<4>(h, nr, s); break;
  }
}

// member tables of every interaction list: record start and inclusive length prefix per member, written
// compacted at the head of the cell's list segment, m_cnt[c] entries.  Members whose record ranges are
// adjacent (Morton-consecutive nonempty cells, common among siblings) are merged into one entry, so the
// interaction kernel issues one TMA bulk copy for the run (merge = 0 keeps one entry per list member).  The
// near field's own leaf is dropped (it is handled by the r2 == 0 pass).
__global__ void member_tables(int64_t n, const int64_t* __restrict__ l_ptr, const int64_t* __restrict__ l_idx,
                              const int64_t* __restrict__ s_ptr, int self_zero, int merge, int upper,
                              int* __restrict__ m_sb, int* __restrict__ m_end, int* __restrict__ m_cnt) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t q0 = l_ptr[c];
  int run = 0, cnt = 0;
  int64_t last_end = -1;
  for (int64_t q = q0; q < l_ptr[c + 1]; q++) {
    const int64_t y = l_idx[q];
    if (self_zero && y == c) continue;
    if (upper && y <= c) continue;  // symmetric kernel: the pair {c, y} belongs to the lower cell
    const int64_t b = s_ptr[y], e = s_ptr[y + 1];
    if (e == b) continue;
    run += (int)(e - b);
    if (merge && cnt > 0 && b == last_end) {
      m_end[q0 + cnt - 1] = run;
    } else {
      m_sb[q0 + cnt] = (int)b;
      m_end[q0 + cnt] = run;
      cnt++;
    }
    last_end = e;
  }
  m_cnt[c] = cnt;
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
  // +1 keeps cells with targets but no sources (they must write zeros); cells without targets cost 0 and are dropped
  const int64_t m = t_ptr[c + 1] - t_ptr[c];
  cost[c] = m > 0 ? (unsigned long long)(m * src) + 1ull : 0ull;
  item[c] = ((int64_t)lev << 40) | c;
}

// symmetric kernel work items: (list, cell) with cost = targets x upper-partner sources (near field: plus the
// leaf's own block)
__global__ void sym_costs(int64_t n, int lst, int near, const int64_t* __restrict__ ptr,
                          const int64_t* __restrict__ l_ptr, const int64_t* __restrict__ l_idx,
                          unsigned long long* __restrict__ cost, int64_t* __restrict__ item,
                          unsigned long long* __restrict__ class_pairs) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int64_t m = ptr[c + 1] - ptr[c];
  int64_t src = near ? m : 0;
  for (int64_t q = l_ptr[c]; q < l_ptr[c + 1]; q++) {
    const int64_t y = l_idx[q];
    if (y > c) src += ptr[y + 1] - ptr[y];
  }
  // sorted descending: M2L items first, then the near field (warps of an SM then mostly run one code path at a
  // time: both together overflow the instruction cache), each by pair count
  const unsigned long long band = near ? 1ull : 2ull;
  cost[c] = (m > 0 && src > 0) ? (band << 56) | ((unsigned long long)(m * src) + 1ull) : 0ull;
  if (m > 0 && src > 0) {  // source passes (64 records) x target chunks of 16 / of 32
    const unsigned long long passes = (unsigned long long)((src + 63) / 64);
    atomicAdd(class_pairs, passes * (unsigned long long)((m + 15) / 16));
    atomicAdd(class_pairs + 1, passes * (unsigned long long)((m + 31) / 32));
  }
  item[c] = ((int64_t)lst << 40) | c;
}

struct SymBuild {
  const int64_t* ptr;
  const int64_t* l_ptr;
  const int* u_cnt;
};

__global__ void make_sym_desc(const int64_t* __restrict__ items, int64_t n, const SymBuild* __restrict__ sb,
                              int4* __restrict__ desc) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t it = items[i];
  const int lst = (int)(it >> 40);
  const int64_t c = it & ((1ll << 40) - 1);
  const SymBuild& B = sb[lst];
  const int64_t tb = B.ptr[c];
  desc[i] = make_int4((int)tb, (int)(B.ptr[c + 1] - tb), (int)B.l_ptr[c], B.u_cnt[c]);
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
      item_costs<<<nblk(Lv.n, 256), 256, 0, s>>>(Lv.n, l, HL.in_ptr.get(), HL.out_ptrd(), Lv.il_ptr.get(),
                                                     Lv.il_idx.get(), cost.get() + off, item.get() + off);
    CKL();
    off += Lv.n;
  }
  {
    const DevLevel& Lv = T.lv[L];
    item_costs<<<nblk(Lv.n, 256), 256, 0, s>>>(Lv.n, L + 1, Lv.t_ptr.get(),
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
  // drop zero-cost items (cells without targets)
  auto hc = to_host(cost_sorted.get(), total, s);
  int64_t nz = 0;
  while (nz < total && hc[nz] > 0) nz++;
  h.n_items = nz;
}

// Symmetric kernel (interact_sym.cuh): upper member tables, work items by descending pair count and their
// descriptors.  Static per H2 matrix.  List ids: 2..L = M2L levels, L + 1 = near field.
void build_sym(DevH2& h, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth;
  h.u_sb.clear();
  h.u_end.clear();
  h.u_cnt.clear();
  h.u_sb.resize(L + 2);
  h.u_end.resize(L + 2);
  h.u_cnt.resize(L + 2);
  std::vector<SymBuild> sb(L + 2);
  std::memset(sb.data(), 0, sizeof(SymBuild) * sb.size());
  std::vector<int> ids;
  for (int l = 2; l <= L; l++) ids.push_back(l);
  ids.push_back(L + 1);
  for (int l : ids) {
    const bool nf = l == L + 1;
    const DevLevel& Lv = T.lv[nf ? L : l];
    const int64_t tot = nf ? Lv.nb_total : Lv.il_total;
    const int64_t* ptr = nf ? Lv.t_ptr.get() : h.lv[l].in_ptr.get();
    h.u_sb[l].alloc(std::max<int64_t>(tot, 1), &h.mem);
    h.u_end[l].alloc(std::max<int64_t>(tot, 1), &h.mem);
    h.u_cnt[l].alloc(std::max<int64_t>(Lv.n, 1), &h.mem);
    if (Lv.n)
      member_tables<<<nblk(Lv.n, 256), 256, 0, s>>>(Lv.n, nf ? Lv.nb_ptr.get() : Lv.il_ptr.get(),
                                                     nf ? Lv.nb_idx.get() : Lv.il_idx.get(), ptr, 0, 1, 1,
                                                     h.u_sb[l].get(), h.u_end[l].get(), h.u_cnt[l].get());
    CKL();
    sb[l].ptr = ptr;
    sb[l].l_ptr = nf ? Lv.nb_ptr.get() : Lv.il_ptr.get();
    sb[l].u_cnt = h.u_cnt[l].get();
  }
  // items, and the pair counts of narrow (<= 16 targets) and wide items
  int64_t total = T.lv[L].n;
  for (int l = 2; l <= L; l++) total += T.lv[l].n;
  DBuf<unsigned long long> cost, cost_sorted, class_pairs;
  DBuf<int64_t> item;
  cost.alloc(std::max<int64_t>(total, 1));
  cost_sorted.alloc(std::max<int64_t>(total, 1));
  item.alloc(std::max<int64_t>(total, 1));
  class_pairs.alloc(2);
  CK(cudaMemsetAsync(class_pairs.get(), 0, 2 * sizeof(unsigned long long), s));
  h.sym_items.alloc(std::max<int64_t>(total, 1), &h.mem);
  int64_t off = 0;
  for (int l : ids) {
    const bool nf = l == L + 1;
    const DevLevel& Lv = T.lv[nf ? L : l];
    if (Lv.n)
      sym_costs<<<nblk(Lv.n, 256), 256, 0, s>>>(Lv.n, l, nf ? 1 : 0, sb[l].ptr, sb[l].l_ptr,
                                                nf ? Lv.nb_idx.get() : Lv.il_idx.get(), cost.get() + off,
                                                item.get() + off, class_pairs.get());
    CKL();
    off += Lv.n;
  }
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, cost.get(), cost_sorted.get(), item.get(),
                                               h.sym_items.get(), total, 0, 64, s));
  DBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(bytes, 1));
  CK(cub::DeviceRadixSort::SortPairsDescending(tmp.get(), bytes, cost.get(), cost_sorted.get(), item.get(),
                                               h.sym_items.get(), total, 0, 64, s));
  auto hc = to_host(cost_sorted.get(), total, s);
  auto cp = to_host(class_pairs.get(), 2, s);
  int64_t nz = 0;
  while (nz < total && hc[nz] > 0) nz++;
  // one chunk width for the whole product (measured: splitting the items over two launches costs more in tail
  // effects than the better width per item saves).  32-target chunks run 12 instead of 16 warps per SM; they
  // pay off when they cut the (chunk, source pass) steps by > 30% AND items are long (many passes per chunk:
  // c1 ~140 steps per item, 6.37 vs 7.38 ms), not for the headline's short items (c2 ~13: 1.63 vs 1.61 ms)
  h.sym_wide = (double)cp[1] < 0.7 * (double)cp[0] && (double)cp[0] > 40.0 * (double)std::max<int64_t>(nz, 1);
  if (getenv("H2B_SETUP_VERBOSE"))
    fprintf(stderr, "[h2b] symmetric kernel: %lld items, %llu (chunk, pass) steps with 16-target chunks, %llu with 32\n",
            (long long)nz, cp[0], cp[1]);
  h.n_sym_items = nz;
  DBuf<SymBuild> dsb;
  dsb.alloc(sb.size());
  CK(cudaMemcpyAsync(dsb.get(), sb.data(), sizeof(SymBuild) * sb.size(), cudaMemcpyHostToDevice, s));
  h.sym_desc.alloc(4 * std::max<int64_t>(nz, 1), &h.mem);
  if (nz)
    make_sym_desc<<<nblk(nz, 256), 256, 0, s>>>(h.sym_items.get(), nz, dsb.get(),
                                                reinterpret_cast<int4*>(h.sym_desc.get()));
  CKL();
  CK(cudaStreamSynchronize(s));
  h.sym_ready = true;
}

// per-list tables of the symmetric kernel (records and outputs change when the scratch is rebuilt)
void build_sym_tabs(DevH2& h, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth;
  std::vector<SymTab> tabs(L + 2);
  std::memset(tabs.data(), 0, sizeof(SymTab) * tabs.size());
  std::vector<int> ids;
  for (int l = 2; l <= L; l++) ids.push_back(l);
  ids.push_back(L + 1);  // the near field (also when the tree has fewer than two levels)
  for (int l : ids) {
    SymTab& t = tabs[l];
    const bool leaf = l > L;
    t.rec = h.pack1.lists[leaf ? std::max(L - 1, 0) : l - 2].get();
    t.ptr = leaf ? T.lv[L].t_ptr.get() : h.lv[l].in_ptr.get();
    t.m_sb = h.u_sb[l].get();
    t.m_end = h.u_end[l].get();
    t.out = leaf ? h.near.get() : h.uin[l].get();
  }
  h.sym_tabs.alloc(sizeof(SymTab) * tabs.size(), &h.mem);
  CK(cudaMemcpyAsync(h.sym_tabs.get(), tabs.data(), sizeof(SymTab) * tabs.size(), cudaMemcpyHostToDevice, s));
}

// Source records (interact.cuh SrcRec) for RHS width nr: allocation, pack
// tables and the static coordinate part.
void build_records(DevH2& h, int nr, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth;
  RecSet& rs = nr == 1 ? h.pack1 : h.pack16;
  const int rsz = 2 * ((T.d + nr + 1) / 2);  // doubles per record
  std::vector<PackTab> pt;
  rs.lists.clear();
  rs.lists.resize(std::max(L - 1, 0) + 1);
  int64_t off = 0;
  auto add = [&](DBuf<double2>& buf, const double* sc, int64_t ld, const double* q, int64_t n) {
    buf.alloc(std::max<int64_t>(n, 1) * rsz / 2, &h.mem);
    PackTab t;
    t.sc = sc;
    t.ld = ld;
    t.q = q;
    t.rec = buf.get();
    t.n = n;
    t.off = off;
    off += n;
    pt.push_back(t);
  };
  for (int l = 2; l <= L; l++) {
    const DevH2Level& HL = h.lv[l];
    add(rs.lists[l - 2], HL.sout_cd(), std::max<int64_t>(HL.out_total, 1), h.wout[l].get(), HL.out_total);
  }
  add(rs.lists[std::max(L - 1, 0)], T.ssd(), T.nq, h.w_sorted.get(), T.nq);
  if (off >= ((int64_t)1 << 31)) throw std::invalid_argument("more than 2^31 source records");
  rs.nlists = (int)pt.size();
  rs.total = off;
  rs.tabs.alloc(sizeof(PackTab) * pt.size(), &h.mem);
  CK(cudaMemcpyAsync(rs.tabs.get(), pt.data(), sizeof(PackTab) * pt.size(), cudaMemcpyHostToDevice, s));
  pack_coords(T.d, h, nr, s);
  CK(cudaStreamSynchronize(s));
}

// list tables (target side + output) for the interaction kernel
void build_tabs(DevH2& h, int64_t R, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth;
  std::vector<LevelTab> tabs(L + 2);
  if (h.m_sb.empty()) {  // member tables (static per H2 matrix)
    h.m_sb.resize(L + 2);
    h.m_end.resize(L + 2);
    h.m_cnt.resize(L + 2);
    const int merge = 1;  // adjacent record ranges merged into one member (one TMA copy per run)
    std::vector<int> ids;
    for (int l = 2; l <= L; l++) ids.push_back(l);
    ids.push_back(L + 1);  // the near field (also when the tree has fewer than two levels)
    for (int l : ids) {
      const bool nf = l == L + 1;
      const DevLevel& Lv = T.lv[nf ? L : l];
      const int64_t tot = nf ? Lv.nb_total : Lv.il_total;
      h.m_sb[l].alloc(std::max<int64_t>(tot, 1), &h.mem);
      h.m_end[l].alloc(std::max<int64_t>(tot, 1), &h.mem);
      h.m_cnt[l].alloc(std::max<int64_t>(Lv.n, 1), &h.mem);
      const int64_t* sp = nf ? (T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get()) : h.lv[l].out_ptrd();
      if (Lv.n)
        member_tables<<<nblk(Lv.n, 256), 256, 0, s>>>(Lv.n, nf ? Lv.nb_ptr.get() : Lv.il_ptr.get(),
                                                         nf ? Lv.nb_idx.get() : Lv.il_idx.get(), sp, nf ? 1 : 0,
                                                         merge, 0, h.m_sb[l].get(), h.m_end[l].get(),
                                                         h.m_cnt[l].get());
      CKL();
    }
  }
  auto rec = [&](const RecSet& rs, int i) -> const double2* { return rs.lists.empty() ? nullptr : rs.lists[i].get(); };
  for (int l = 0; l <= L + 1; l++) {
    LevelTab& t = tabs[l];
    std::memset(&t, 0, sizeof t);
    if (l >= 2 && l <= L) {
      const DevLevel& Lv = T.lv[l];
      const DevH2Level& HL = h.lv[l];
      t.tc = HL.tin_c.get();
      t.ld_t = std::max<int64_t>(HL.in_total, 1);
      t.t_ptr = HL.in_ptr.get();
      t.s_ptr = HL.out_ptrd();
      t.rec1 = rec(h.pack1, l - 2);
      t.rec16 = rec(h.pack16, l - 2);
      t.l_ptr = Lv.il_ptr.get();
      t.l_idx = Lv.il_idx.get();
      t.m_sb = h.m_sb[l].get();
      t.m_end = h.m_end[l].get();
      t.m_cnt = h.m_cnt[l].get();
      t.out = h.uin[l].get();
    } else if (l == L + 1) {
      const DevLevel& Lv = T.lv[L];
      t.tc = T.tsd();
      t.ld_t = T.np;
      t.t_ptr = Lv.t_ptr.get();
      t.s_ptr = T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get();
      t.rec1 = rec(h.pack1, std::max(L - 1, 0));
      t.rec16 = rec(h.pack16, std::max(L - 1, 0));
      t.l_ptr = Lv.nb_ptr.get();
      t.l_idx = Lv.nb_idx.get();
      t.m_sb = h.m_sb[L + 1].get();
      t.m_end = h.m_end[L + 1].get();
      t.m_cnt = h.m_cnt[L + 1].get();
      t.out = h.near.get();
    }
  }
  h.tabs.alloc(sizeof(LevelTab) * tabs.size(), &h.mem);
  CK(cudaMemcpyAsync(h.tabs.get(), tabs.data(), sizeof(LevelTab) * tabs.size(), cudaMemcpyHostToDevice, s));
  if (!h.item_desc.n) {
    h.item_desc.alloc(4 * std::max<int64_t>(h.n_items, 1), &h.mem);
    if (h.n_items)
      make_item_desc<<<nblk(h.n_items, 256), 256, 0, s>>>(h.items.get(), h.n_items,
                                                          reinterpret_cast<const LevelTab*>(h.tabs.get()),
                                                          reinterpret_cast<int4*>(h.item_desc.get()));
    CKL();
  }
  CK(cudaStreamSynchronize(s));
}

void ensure_scratch(DevH2& h, int64_t R, cudaStream_t s) {
  const DevTree& T = *h.t;
  if (h.scratch_nrhs == R) return;
  // another RHS width: park the active set (at most 3 parked, oldest dropped) and revive a parked one of width R
  MatvecScratch& act = static_cast<MatvecScratch&>(h);
  if (h.scratch_nrhs != 0) {
    h.parked.push_back(std::move(act));
    act = MatvecScratch();
    if (h.parked.size() > 3) h.parked.erase(h.parked.begin());
  }
  for (auto it = h.parked.begin(); it != h.parked.end(); ++it)
    if (it->scratch_nrhs == R) {
      act = std::move(*it);
      h.parked.erase(it);
      return;
    }
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
  // the one-directional kernel (multi-RHS chunks, non-symmetric operators) needs its work list and member
  // tables; a symmetric operator applied to single vectors never builds them
  const bool need_dir = !h.symmetric || R >= 16;
  if (need_dir && !h.items.n) build_items(h, s);
  if (!h.work_counter.n) h.work_counter.alloc(1, &h.mem);
  if (h.own_in.empty()) {
    h.own_in.resize(T.depth + 1);
    h.own_out.resize(T.depth + 1);
    for (int l = 2; l <= T.depth; l++) {
      const DevH2Level& HL = h.lv[l];
      h.own_in[l].alloc(std::max<int64_t>(HL.in_total, 1), &h.mem);
      fill_owner<<<nblk(HL.n, 256), 256, 0, s>>>(HL.n, HL.in_ptr.get(), h.own_in[l].get());
      CKL();
      if (!h.symmetric) {
        h.own_out[l].alloc(std::max<int64_t>(HL.out_total, 1), &h.mem);
        fill_owner<<<nblk(HL.n, 256), 256, 0, s>>>(HL.n, HL.out_ptrd(), h.own_out[l].get());
        CKL();
      }
    }
    // compact transfer operators (transfer.cuh): rows of a cell = its children's stacked pivots, at the leaves
    // its points
    h.c_in.clear();
    h.c_out.clear();
    h.c_in.resize(T.depth + 1);
    if (!h.symmetric) h.c_out.resize(T.depth + 1);
    for (int l = 2; l <= T.depth; l++) {
      const DevLevel& Lv = T.lv[l];
      const DevH2Level& HL = h.lv[l];
      const bool leaf = l == T.depth;
      const int64_t* in_base = leaf ? Lv.t_ptr.get() : h.lv[l + 1].in_ptr.get();
      const int64_t in_space = leaf ? T.np : h.lv[l + 1].in_total;
      build_compact(h.c_in[l], HL.n, HL.in_total, HL.in_ptr.get(), HL.m_in.get(), HL.pmat.get(), HL.pm_off.get(),
                    in_base, leaf ? nullptr : Lv.ch_ptr.get(), in_space, true, h.symmetric != 0, &h.mem, s);
      if (!h.symmetric) {
        const int64_t* out_base = leaf ? (T.shared ? Lv.t_ptr.get() : Lv.s_ptr.get()) : h.lv[l + 1].out_ptrd();
        const int64_t out_space = leaf ? T.nq : h.lv[l + 1].out_total;
        build_compact(h.c_out[l], HL.n, HL.out_total, HL.out_ptrd(), HL.n_outd(), HL.qmatd(), HL.qm_offd(), out_base,
                      leaf ? nullptr : Lv.ch_ptr.get(), out_space, false, true, &h.mem, s);
      }
    }
  }
  h.pack1 = RecSet();
  h.pack16 = RecSet();
  if (R >= 16) build_records(h, 16, s);
  if (R % 16) build_records(h, 1, s);
  if (need_dir) build_tabs(h, R, s);
  if (h.symmetric && R % 16) {
    if (!h.sym_ready) build_sym(h, s);
    build_sym_tabs(h, s);
  }
  h.scratch_nrhs = R;
}

// RHS widths supported by the interaction kernel
void rhs_chunks(int64_t R, std::vector<std::pair<int64_t, int>>& out) {
  out.clear();
  int64_t r0 = 0;
  while (r0 < R) {
    int64_t left = R - r0;
    int nr = left >= 16 ? 16 : 1;  // instantiated widths: 16 and 1
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
  // gather, P2M, M2M x (L-2), interaction launches per RHS chunk, L2L x (L-2), L2P+scatter.  Per chunk: a record
  // pack unless one RHS (the gather and the upward pass write the records), then the interaction kernel (one
  // launch)
  const bool sym = h.symmetric && h.sym_ready && (nrhs % 16) != 0;
  int64_t inter = 0;
  for (auto& c : ch) {
    inter += nrhs == 1 ? 0 : 1;
    inter += (sym && c.second == 1) ? (h.n_sym_items > 0) : 1;
  }
  if (L < 2) return 1 + inter + 1;
  return 1 + 1 + (L - 2) + inter + (L - 2) + 1;
}

void matvec(DevH2& h, const double* w, double* u, int64_t R, cudaStream_t s) {
  const DevTree& T = *h.t;
  const int L = T.depth, d = T.d;
  ensure_scratch(h, R, s);
  h.last_nrhs = R;
  KParams kp = make_kp(h.kind, h.a);
  std::vector<std::pair<int64_t, int>> chunks;
  rhs_chunks(R, chunks);
  cudaEvent_t ev[5];
  if (g_profile) {
    for (auto& e : ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ev[0], s));
  }
  // one RHS: the gather and the upward pass also write the records' charge slots (pack_records skipped)
  const bool fused_pack = R == 1 && !h.pack1.lists.empty();
  const int rs1 = 2 * ((T.d + 2) / 2);  // doubles per NR = 1 record
  auto recq = [&](int list) -> double* {
    return fused_pack ? reinterpret_cast<double*>(h.pack1.lists[list].get()) + T.d : nullptr;
  };
  // symmetric one-RHS product: the interaction kernel accumulates into zeroed u_in / near buffers; with one RHS
  // the gather and the upward pass clear them in passing (same index spaces), otherwise memsets do
  const bool sym = h.symmetric && h.sym_ready && (R % 16) != 0;
  const bool fused_zero = sym && R == 1 && T.shared && L >= 2;
  gather_rows<<<nblk(T.nq * R, 256), 256, 0, s>>>(w, T.sperm(), T.nq, R, h.w_sorted.get(),
                                                  recq((int)h.pack1.lists.size() - 1), rs1,
                                                  fused_zero ? h.near.get() : nullptr);
  CKL();
  if (L >= 2) {
    // ---- upward pass: P2M at the leaves, then M2M (one or a few threads per output row) ----
    auto own_out = [&](int l) { return h.symmetric ? h.own_in[l].get() : h.own_out[l].get(); };
    auto c_up = [&](int l) -> const CompactOps& { return h.symmetric ? h.c_in[l] : h.c_out[l]; };
    {
      const DevH2Level& HL = h.lv[L];
      launch_up(c_up(L), HL.out_total, own_out(L), HL.out_ptrd(), h.w_sorted.get(), h.wout[L].get(), R, s,
                recq(L - 2), rs1, fused_zero ? h.uin[L].get() : nullptr);
    }
    for (int l = L - 1; l >= 2; l--) {
      const DevH2Level& HL = h.lv[l];
      launch_up(c_up(l), HL.out_total, own_out(l), HL.out_ptrd(), h.wout[l + 1].get(), h.wout[l].get(), R, s,
                recq(l - 2), rs1, fused_zero ? h.uin[l].get() : nullptr);
    }
  }
  if (g_profile) CK(cudaEventRecord(ev[1], s));
  // ---- every M2L level + the near field in one launch per RHS chunk ----
  // one-RHS chunks on the symmetric path: each unordered cell pair evaluated once (interact_sym.cuh), results
  // accumulated with FP64 reductions into zeroed u_in / near buffers
  if (sym && !fused_zero) {
    for (int l = 2; l <= L; l++)
      CK(cudaMemsetAsync(h.uin[l].get(), 0, sizeof(double) * h.lv[l].in_total * R, s));
    CK(cudaMemsetAsync(h.near.get(), 0, sizeof(double) * T.np * R, s));
  }
  for (auto& ch : chunks) {
    if (sym && ch.second == 1) interact_sym_all(d, h.kind, h, R, ch.first, kp, s);
    else interact_all(d, h.kind, h, R, ch.first, ch.second, kp, s);
  }
  if (g_profile) CK(cudaEventRecord(ev[2], s));
  // ---- downward pass (L2L): one thread (upper levels: a few lanes) per general child row, one per pivot ----
  for (int l = 2; l < L; l++)
    launch_down<false>(h.c_in[l], h.lv[l].in_total, h.lv[l].in_ptr.get(), h.uin[l].get(), h.uin[l + 1].get(), nullptr,
                       nullptr, R, s);
  if (g_profile) CK(cudaEventRecord(ev[3], s));
  // ---- L2P + near field, scattered to the caller's order ----
  if (L >= 2)
    launch_down<true>(h.c_in[L], h.lv[L].in_total, h.lv[L].in_ptr.get(), h.uin[L].get(), u, h.near.get(),
                      T.t_perm.get(), R, s);
  else
    scatter_near<<<nblk(T.np * R, 256), 256, 0, s>>>(T.np, h.near.get(), T.t_perm.get(), u, R);
  CKL();
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
// dense oracles (matvec.py:233 dense_matvec) and kernel blocks
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
