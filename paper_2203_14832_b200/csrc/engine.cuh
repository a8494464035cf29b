// engine.cuh — device-resident tree and H2 representation.
//
// HBM layout (all arrays device memory, owned by the structs below):
//   * points: original row-major P, Q (for gathers by global index) plus
//     Morton-sorted SoA copies  ts[k*np + i]  (k = coordinate) so a leaf's
//     points are one contiguous, coalesced range.
//   * cells: per level, nonempty cells in Morton order.  A cell's points are
//     [t_ptr[c], t_ptr[c+1]) of the sorted arrays and its children are the
//     contiguous range [ch_ptr[c], ch_ptr[c+1]) of the next level — so every
//     M2M/L2L operand is a contiguous slice.
//   * lists: neighbour / interaction lists in CSR, each list sorted by the
//     reference's row-major multi-index key (geometry.py:333-334) because the
//     order of the ACA candidate columns depends on it.
//   * H2: per level, pivot coordinates (SoA), pivot global indices, and the
//     interpolation operators of every cell, column-major (row index
//     fastest) at tight per-cell offsets.
#pragma once
#include <memory>
#include <vector>

#include "common.cuh"

namespace h2b {

struct DevLevel {
  int64_t n = 0;
  DBuf<unsigned long long> code;  // Morton prefix at this level
  DBuf<int64_t> rmkey;            // reference row-major key
  DBuf<int64_t> t_ptr, s_ptr;     // n+1
  DBuf<int64_t> parent;           // n (index in level-1)
  DBuf<int64_t> ch_ptr;           // n+1 (range in level+1)
  DBuf<int64_t> nb_ptr, nb_idx, il_ptr, il_idx;
  DBuf<int64_t> rm_perm;  // reference-order position -> internal index
  DBuf<int64_t> rm_inv;   // internal index -> reference-order position
  int64_t nb_total = 0, il_total = 0;
};

struct DevTree {
  int d = 0, depth = 0, shared = 0, over_capacity = 0, Lmax = 0;
  int64_t np = 0, nq = 0, nu = 0;
  double eta = 0, half = 0, mid[H2B_MAXD] = {0}, lo0[H2B_MAXD] = {0};
  MemStats mem;
  DBuf<double> P, Q;          // row-major originals (Q aliases P when shared)
  DBuf<double> ts, ss;        // sorted SoA
  DBuf<int64_t> t_perm, s_perm;  // sorted position -> original index
  std::vector<DevLevel> lv;
  const double* Pd() const { return P.get(); }
  const double* Qd() const { return shared ? P.get() : Q.get(); }
  const double* tsd() const { return ts.get(); }
  const double* ssd() const { return shared ? ts.get() : ss.get(); }
  const int64_t* sperm() const { return shared ? t_perm.get() : s_perm.get(); }
  const DevLevel& L(int l) const { return lv[l]; }
};

struct DevH2Level {
  int64_t n = 0;
  DBuf<int64_t> kin, kout, in_ptr, out_ptr;  // out aliases in when symmetric
  DBuf<int64_t> t_in, s_in, t_out, s_out;    // global indices
  DBuf<double> tin_c, sout_c;                // pivot coordinates, SoA with ld = in_total/out_total
  DBuf<int64_t> m_in, n_out;                 // rows of the row / column interpolator
  DBuf<int64_t> pm_off, qm_off;              // per-cell offsets into pmat / qmat
  DBuf<double> pmat, qmat;                   // column-major (rows fastest)
  DBuf<int64_t> nevals, conv;
  int64_t in_total = 0, out_total = 0;
  const int64_t* koutd() const { return kout.n ? kout.get() : kin.get(); }
  const int64_t* out_ptrd() const { return out_ptr.n ? out_ptr.get() : in_ptr.get(); }
  const double* sout_cd() const { return sout_c.n ? sout_c.get() : tin_c.get(); }
  const double* qmatd() const { return qmat.n ? qmat.get() : pmat.get(); }
  const int64_t* qm_offd() const { return qm_off.n ? qm_off.get() : pm_off.get(); }
  const int64_t* n_outd() const { return n_out.n ? n_out.get() : m_in.get(); }
};

// Compact transfer operators of one level and side (transfer.cuh): the interpolators without their identity
// (pivot) rows.
struct CompactOps {
  DBuf<int> piv_pos;      // per pivot: row position of its identity row in the level's row space, -1 = dense cell
  DBuf<int64_t> g_ptr;    // n + 1: general-row prefix per cell
  DBuf<int> g_pos;        // per general row: its row position
  DBuf<int> g_owner;      // per general row: its cell
  DBuf<int64_t> op_off;   // n + 1: offset of the cell's g x k block
  DBuf<double> op_dn;     // [s * g + j] (downward: thread per general row)
  DBuf<double> op_up;     // [j * k + s] (upward: thread per pivot)
  int64_t g_total = 0, op_total = 0;
  int sg_up = 1, sg_dn = 1;  // lanes per output row
};

// Packed source records of every interaction source list for one RHS width
// (interact.cuh SrcRec): per level the outgoing pivots, then the leaf points.
struct RecSet {
  std::vector<DBuf<double2>> lists;  // [0, L - 2]: levels 2..L; [L - 1]: near field
  DBuf<unsigned char> tabs;          // PackTab per list
  int nlists = 0;
  int64_t total = 0;
};

// Matvec scratch of one right-hand-side width: everything whose size or device pointers depend on nrhs.  The
// active set lives in DevH2 (base class); sets of other widths are parked in DevH2::parked, so alternating
// widths (e.g. a 16-RHS block product between single-vector products) does not rebuild the source records.
struct MatvecScratch {
  int64_t scratch_nrhs = 0;
  DBuf<double> w_sorted;
  std::vector<DBuf<double>> wout, uin;
  DBuf<double> near;        // near-field sums (sorted target order)
  DBuf<unsigned char> tabs; // per-list pointer tables for the interaction kernel
  RecSet pack1, pack16;     // source records for RHS chunks of width 1 / 16
  DBuf<unsigned char> sym_tabs;
};

struct DevH2 : MatvecScratch {
  const DevTree* t = nullptr;
  int kind = 0, symmetric = 1;
  double a = 0, eps = 0;
  MemStats mem;
  std::vector<DevH2Level> lv;  // indexed by level; levels < 2 empty
  int64_t evals_pivots = 0, evals_couplings = 0, evals_nearfield = 0, max_rank = 0, cells_visited = 0;
  int64_t setup_ns = 0, unconverged = 0;
  int64_t last_nrhs = 0;  // RHS width of the last product (its coefficient vectors are still in wout / uin)
  // matvec scratch of other RHS widths (most recently used last; at most 3 parked)
  std::vector<MatvecScratch> parked;
  DBuf<double> io_w, io_u;  // device staging for host-pointer calls
  DBuf<int64_t> items;      // interaction work list ((list << 40) | cell), by descending pair count
  int64_t n_items = 0;
  DBuf<int> item_desc;      // per work item {first target, targets, list begin, list end} (int4)
  std::vector<DBuf<int>> own_in, own_out;  // per level: pivot position -> owning cell
  std::vector<CompactOps> c_in, c_out;      // per level: compact row / column interpolators (c_out empty when symmetric)
  std::vector<DBuf<int>> m_sb, m_end, m_cnt;       // per interaction list: member tables (interact.cuh LevelTab)
  DBuf<unsigned long long> work_counter;    // persistent interaction kernel: next work item
  // symmetric one-RHS interaction kernel (interact_sym.cuh): upper member tables per list (partners Y > X),
  // work items (list, cell) by descending pair count, descriptors and per-list tables
  std::vector<DBuf<int>> u_sb, u_end, u_cnt;
  DBuf<int64_t> sym_items;
  DBuf<int> sym_desc;
  int64_t n_sym_items = 0;
  bool sym_wide = false;  // 32-target chunks (most pairs in items with > 16 targets) instead of 16
  bool sym_ready = false;
};

// tree.cu
std::unique_ptr<DevTree> build_tree(const double* P, int64_t np, const double* Q, int64_t nq, int d, int shared,
                                    int64_t nu, double eta, bool on_device, cudaStream_t s);
// nnca.cu
std::unique_ptr<DevH2> assemble(const DevTree& t, int kind, double a, double eps, bool force_general,
                                int64_t max_rank, cudaStream_t s);
void release_workspace();  // frees the per-device ACA arenas
void aca_single(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d, double eps,
                int64_t cap, double* U, double* V, int64_t* rp, int64_t* cp, int* conv, int64_t* nevals,
                int64_t* rank);
// matvec.cu
void matvec(DevH2& h, const double* w, double* u, int64_t nrhs, cudaStream_t s);
void prepare_matvec(DevH2& h, cudaStream_t s);
int64_t matvec_launches(const DevH2& h, int64_t nrhs);
void set_profiling(bool on);
double fp64_peak_tflops(cudaStream_t s);
void last_stage_ms(double* ms5);
void dense_matvec(int kind, double a, const double* P, int64_t np, const double* Q, int64_t nq, int d,
                  const double* w, double* u, int64_t nrhs, cudaStream_t s);
void kernel_block(int kind, double a, const double* X, int64_t m, const double* Y, int64_t n, int d, double* out,
                  cudaStream_t s);

}  // namespace h2b
