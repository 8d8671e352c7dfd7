// Internal data structures shared by the host symbolic analysis (symbolic.cpp) and the
// device numeric phase (numeric.cu).  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#ifdef __CUDACC__
#define SGN_HD __host__ __device__ __forceinline__
#else
#define SGN_HD inline
#endif

namespace sgn {

constexpr int kTile = 32;   // assembly tile, panel width, update tile
constexpr int kPanelTiles = 4;   // 32-row tiles per panel CTA (one per warp)

// One dense front (supernode) of the multifrontal assembly tree.
struct Front {
  int64_t first = 0;      // first elimination position of its pivots
  int32_t npiv = 0;       // fully-summed (pivot) unknowns
  int32_t nrow = 0;       // npiv + |struct|
  int32_t parent = -1;
  int32_t level = 0;      // height: leaves 0, parent = 1 + max(children)
  int32_t pivtype = 1;    // 1: 1x1 pivots, 2: 2x2 (x_i, lambda_j) pair pivots
  int32_t is_root_p = 0;  // the dense p front (skipped by SGN_SOLVE_LEADING)
  int32_t child_begin = 0, child_end = 0;  // range in Symbolic::children
  int64_t foff = 0;       // offset of the nrow x nrow column-major front (doubles)
  int64_t srow_off = 0;   // offset of struct rows (positions) in Symbolic::srows
  int64_t rel_off = 0;    // offset of rel map (struct -> parent local rows)
  int64_t uoff = 0;       // offset of the forward-solve update vector (nstruct)
  int64_t woff = 0;       // offset of its rel ranges per parent tile (Symbolic::reltile)
  int64_t voff = 0;       // offset of the solve front vector (nrow)
  int64_t tile_base = 0;  // first assembly tile id
  int64_t zoff = 0;       // offset of the solve panel Z = [I; L21] L11^{-1} (nrow x npiv)
  int64_t doff = 0;       // offset of the factored 32x32 diagonal blocks (scratch)
  int64_t cbase = 0;      // first dependency counter of the front (persistent factorization)
  int32_t ftotal = 0;     // assembly + panel + update tasks of the front
  int32_t noz = 0;        // no solve panel: the root p-front of a large n_p (blocked substitution)
};

// Device-side mirror of Front (POD, 16-byte aligned for vector loads).
struct DFront {
  int64_t first;
  int64_t foff;
  int64_t srow_off;
  int64_t rel_off;
  int64_t uoff;
  int64_t woff;
  int64_t voff;
  int64_t tile_base;
  int64_t zoff;
  int64_t doff;
  int32_t npiv, nrow, parent, pivtype;
  int32_t child_begin, child_end, is_root_p, level;
  int64_t cbase;
  int32_t ftotal, flags;  // flags bit 0: noz (Front::noz)
};

// Leading dimension of a front's dense storage and of its solve panel Z: nrow rounded up to
// even, so every column starts 16-byte aligned (the cp.async operand staging of the 64x64
// DMMA blocks, factor_dag.cu:f_block64).
SGN_HD int64_t front_ld(int nrow) { return (int64_t)nrow + (nrow & 1); }

// Split tile grid of a front: pivot tiles a < P cover rows [32a, min(32a+32, npiv)), the
// contribution tiles a >= P cover [npiv + 32(a-P), ...).  Pivot step k is tile k, so every
// Schur-update step touches whole tiles and per-tile dependency counters are exact.
SGN_HD int ptiles(int npiv) { return (npiv + 31) / 32; }
SGN_HD int ntiles_front(int npiv, int nrow) { return ptiles(npiv) + (nrow - npiv + 31) / 32; }
SGN_HD int tile_lo(int npiv, int a) {
  const int P = ptiles(npiv);
  return a < P ? 32 * a : npiv + 32 * (a - P);
}
SGN_HD int tile_hi(int npiv, int nrow, int a) {
  const int P = ptiles(npiv);
  return a < P ? (32 * a + 32 < npiv ? 32 * a + 32 : npiv) : (npiv + 32 * (a - P) + 32 < nrow ? npiv + 32 * (a - P) + 32 : nrow);
}
SGN_HD int tile_of_row(int npiv, int r) { return r < npiv ? r / 32 : ptiles(npiv) + (r - npiv) / 32; }

// Persistent factorization task (16 bytes).  kind_k = kind | (k << 3); waits and signals
// are derived from the coordinates on the device (no stored wait lists).  Per pivot step
// k of a front the diagonal block D_k is factored ONCE (by the assembly task of tile
// (0,0) for k = 0, else by F_DIAGUPD(k-1)) and published to scratch as [D | L^T | D^-1]:
//   F_ASM     (f, a=ti, b=tj): waits DONE(child) == ftotal(child) for every child; k = 1: the
//                              64x64 block {ti, ti+1} x {tj, tj+1} (its lower tiles)
//   F_PANEL   (f, k, a=t)    : TRSM of row tiles {k+1} (t = 0) or k+2+4(t-1).. (t >= 1);
//                              waits DIAG(f, k), TILE(f, i, k) == 1 + k for its rows
//   F_UPDATE  (f, k, a=ti, b=tj): waits PAN(f, k) == TRSM tasks of step k, TILE(f,ti,tj) == 1+k
//   F_DIAGUPD (f, k)         : last update of tile (k+1, k+1) + LDL^T of D_{k+1}; waits as
//                              F_UPDATE(k, k+1, k+1); signals DIAG(f, k+1)
//   F_ZPANEL  (f, a=t, b=cb)  : solve-panel block Z(t, cb) = sum_j L(t, j) Z(j, cb) (+ left solve
//                              with L(t, t) for pivot tiles).  Waits DIAG(f, t) (pivot tiles) or
//                              PAN(f, P-1) (struct tiles), then progressively, per term j,
//                              ZC(f, cb) > j - cb; pivot tiles signal ZC(f, cb)
// counters of front f at cbase: DONE, PAN(k), DIAG(k) (k < P), TILE(ti*(ti+1)/2 + tj), ZC(cb),
// PANT(k, t) (k < P, t < T)
//   F_FAT     (f, a, b)      : a whole small front in one CTA: runs fat[a .. b) (its tasks in the
//                              order above, then its Z blocks) back to back; the sub-tasks signal
//                              their own counters, so the waits between them pass at once
//   F_UPD2    (f, k, a=ti, b=tj | ns << 16 [| 0x8000: one column tile, 64x32]): the update of the 64x64 block of tiles
//                              {ti, ti+1} x {tj, tj+1} (tiles past the front or above the
//                              diagonal skipped): waits and signals as F_UPDATE per tile
//   F_ZPAN2   (f, a=t, b=cb)  : struct-tile solve-panel blocks Z({t, t+1}, {cb, cb+1}) (t >= P) in
//                              one 64x64 DMMA product; waits PAN(P-1) and the complete Z
//                              columns ZC(cb), ZC(cb+1); signals nothing (read by the solve)
enum FKind : int32_t { F_ASM = 0, F_PANEL = 1, F_UPDATE = 2, F_ZPANEL = 3, F_DIAGUPD = 4, F_FAT = 5, F_UPD2 = 6,
                       F_ZPAN2 = 7 };
struct FTask { int32_t kind_k, f, a, b; };
constexpr int kDiagStride = 2 * kTile * kTile + 3 * kTile;   // scratch per step: D, L^T, D^-1
SGN_HD int panel_tasks(int npiv, int nrow, int k) {   // TRSM tasks of step k
  const int T = ntiles_front(npiv, nrow);
  const int rest = T - k - 2;
  return (k + 1 < T ? 1 : 0) + (rest > 0 ? (rest + 3) / 4 : 0);
}
SGN_HD int cnt_pan(int k) { return 1 + k; }
SGN_HD int cnt_diag(int P, int k) { return 1 + P + k; }
SGN_HD int cnt_tile(int P, int ti, int tj) { return 1 + 2 * P + ti * (ti + 1) / 2 + tj; }
SGN_HD int cnt_zc(int P, int T, int slab) { return 1 + 2 * P + T * (T + 1) / 2 + slab; }
// PANT(k, t): TRSM task t of step k (t = 0: row tile k+1; t >= 1: row tiles k+2+4(t-1)..).
// A Schur update of step k waits for the tasks of its two row tiles only (earlier steps of
// those rows are implied: each TRSM waited for its rows' updates of the previous step).
SGN_HD int cnt_pant(int npiv, int nrow, int k, int t) {
  const int P = ptiles(npiv), T = ntiles_front(npiv, nrow);
  return 1 + 2 * P + T * (T + 1) / 2 + (nrow + 31) / 32 + k * T + t;
}
SGN_HD int pan_task_of(int k, int tile) { return tile == k + 1 ? 0 : 1 + (tile - k - 2) / 4; }
// PAN0(k): the TRSM task of row tile k+1 (t = 0) of step k -- all the diagonal update reads
SGN_HD int cnt_pan0(int npiv, int nrow, int k) { return cnt_pant(npiv, nrow, k, 0); }

struct Work { int32_t f, a, b, c; };   // generic work item

enum LaunchKind : int32_t { L_ASM = 0, L_PANEL = 1, L_UPDATE = 2, L_ZPANEL = 3 };
constexpr int kFwdRows = 32;    // rows per CTA of the forward-solve GEMV
constexpr int kFwdCols = 64;    // pivot columns of a one-task ("fat") forward front solve
constexpr int kFwdChunk = 128;  // columns (K chunk) per CTA of the tiled forward-solve GEMV
constexpr int kBwdCols = 32;    // columns per CTA of the backward-solve dots
constexpr int kBwdRows = 256;   // rows (K chunk) per CTA of the backward-solve dots (two 128-row halves)
constexpr int kFatRows = 512;     // rows of a one-task ("fat") forward front solve
constexpr int kFatRowsBwd = 128;  // rows of a one-task backward front solve (Z prefetched whole)
// Persistent dependency-driven (DAG) schedule: a task runs after every (counter, target)
// wait in waits[w0, w1) is met, then bumps counter `sig` (-1: none).  Tasks are listed in a
// topological order and grabbed in that order by resident CTAs, so waits always target
// earlier tasks and the schedule cannot deadlock.
// T_FWD_FAT / T_BWD_FAT: the whole forward / backward step of a small front in one task
// T_RFWD / T_RBWD: row tile j of a no-Z root front (work item a = -2 - j), blocked
// substitution with L11 read from the front, progressive over the front's own counter
enum TaskKind : int32_t { T_FWD = 1, T_BWD = 2, T_FWD_FAT = 3, T_BWD_FAT = 4, T_RFWD = 5, T_RBWD = 6 };
struct Task { int32_t kind, f, a, b, c, sig, w0, w1; };
struct Launch { int32_t kind; int32_t level; int64_t off; int64_t count; int32_t pivtype = 1; int32_t pad = 0; };

// Options of the symbolic analysis and its schedules (mirror of sgn_symbolic_options).
struct SymOptions {
  int32_t leaf_size = 64;     // max unknowns in a leaf front
  int32_t p_order = 0;        // 0: p unknowns last (dense root front); 1: p pairs in the dissection
  int32_t upd_group = 8;      // pivot steps per grouped Schur-update task
  int32_t zinline = 8;        // fronts with >= zinline pivot tiles build Z inline
  int32_t zquota = 256;       // queued Z blocks interleaved per pivot step
  int32_t noz_tiles = 0;      // root p-front of >= noz_tiles tiles gets no Z (0: off)
  int32_t fat_tiles = 0;      // fronts of <= fat_tiles tiles factor as one task (0: off)
  int32_t fat_solve = 1;      // small fronts solve as one task
  int32_t generic_pairs = 1;  // generic mode: 2x2 pivots on consecutive unknowns
  int32_t upd_pair = 31;      // grouped Schur updates on 64x64 blocks (F_UPD2); bit 1: struct-tile
                              // Z blocks on 64x64 blocks too (F_ZPAN2); bit 2: assembly
                              // on 64x64 blocks (F_ASM, k = 1); bit 3: single-column updates
                              // (look-ahead, single-step, unpaired groups) as row pairs
                              // (F_UPD2 with b bit 15, 64x32); bit 4: look-ahead column k + 1 and
                              // single-step column k + 2 of step k as one 64x64 block per row pair
                              // below the chain rows; default 31 = all
  int32_t pair_min_tiles = 0; // bits 0-1 apply to fronts of >= this many tiles (0: auto)
  int32_t upd_group_cb = 32;  // pivot steps per grouped update of contribution-block columns
  int32_t defer_groups = 1;   // grouped updates of step k listed after the panels / diagonal update of step k + 1
  int32_t zdist = 2;          // queued Z blocks of fronts at levels <= lv - zdist are interleaved into level lv
};

struct Symbolic {
  int64_t n = 0, n_x = 0, n_p = 0, n_c = 0;
  bool pair_mode = false;
  int32_t p_order = 0;                         // SymOptions::p_order in effect
  std::vector<int64_t> indptr, indices;       // input full CSC pattern
  std::vector<int64_t> perm, ipos;             // perm[pos] = unknown; ipos[unknown] = pos
  std::vector<Front> fronts;                   // postorder (children before parents)
  std::vector<int32_t> children;
  std::vector<int64_t> srows;                  // struct rows (positions), sorted per front
  std::vector<int32_t> rel;                    // per front: struct row -> parent local row
  std::vector<int32_t> reltile;                // per front: first rel index >= each parent tile (T_parent + 1)
  std::vector<int8_t> kind_pos;                // 0 none, 1 +eps_x, 2 -eps_lambda
  std::vector<int32_t> front_of_pos;
  // assembly entry lists per tile
  std::vector<int64_t> tile_ptr;               // ntiles+1
  std::vector<int64_t> tile_nnz;               // K nnz index
  std::vector<int32_t> tile_loc;               // (lr%32)*32 + (lc%32)
  int64_t ntiles = 0;
  // schedule
  int32_t n_levels = 0;
  std::vector<std::vector<int32_t>> level_fronts;
  std::vector<int64_t> level_task_off;         // first factorization task of each level (ftasks index)
  std::vector<Work> work;                      // all work items
  std::vector<Launch> launches;                // factorization launch schedule
  // solve work lists per level (items into `work`): forward (f, row0), backward (f, col0)
  std::vector<int64_t> fwd_off, fwd_cnt, bwd_off, bwd_cnt, gat_off, gat_cnt;
  std::vector<int32_t> lvl_max_piv;
  // chunk-split groups: per (front, tile) group -> number of chunks, partial-sum base
  std::vector<int32_t> grp_nchunk;
  std::vector<int64_t> grp_base;
  int64_t n_groups = 0, part_doubles = 0;
  // persistent solve schedule: tasks, flat (counter, target) wait pairs, counter count
  std::vector<Task> stasks;
  std::vector<int32_t> swaits;
  int32_t n_scnt = 0;
  // inverse extend-add map for the solve: front row (voff + r) -> children update slots
  // (ubuf offsets) in child order: v[r] = b[r] + sum u[gsrc[gptr[voff+r] .. gptr[voff+r+1])]
  std::vector<int64_t> gptr;
  std::vector<int32_t> gsrc;
  // persistent factorization: tasks in topological order + counters per instance
  std::vector<FTask> ftasks;
  std::vector<FTask> fat;                      // sub-tasks of the F_FAT fronts
  int64_t n_fcnt = 0;
  // sizes
  int64_t front_doubles = 0, u_doubles = 0, w_doubles = 0, v_doubles = 0, z_doubles = 0, d_doubles = 0;
  int64_t nnz_l = 0; double flops = 0; int64_t max_front = 0, max_piv = 0;
};

// arguments of the persistent factorization launch (factor_dag.cu); head is followed by
// batch x n_fcnt dependency counters, all zeroed before every factorization
struct FactorArgs {
  const FTask* tasks; int64_t ntask; int32_t batch; const FTask* fat;
  int* head; int* cnt; int64_t n_fcnt;
  const DFront* fronts; const int32_t* children; const int32_t* rel; const int32_t* reltile;
  const int64_t* tile_ptr; const int64_t* tile_nnz; const int32_t* tile_loc; const int8_t* kind_pos;
  const double* values; int64_t vstride; double eps_x, eps_l; const double* eps_xv; const double* eps_lv;
  const int64_t* perm; double* fstore; int64_t fstride; double* zstore; int64_t zstride;
  double* dscr; int64_t dstride; long long* status;
  unsigned long long* trace;   // optional (SGN_FDAG_TRACE=1): 4 words per task
  int32_t run;                 // instances per grab (divides batch; 1 for a single instance)
  // CTAs with blockIdx >= retire_from leave once a task index >= retire_at has been reached
  // (sgn_factor_set_retire): a concurrent launch takes over their SM slots for the
  // dependency-bound top levels
  int32_t retire_from; int64_t retire_at;
};
int factor_dag_grid();   // persistent CTAs: SMs x occupancy limit
int min_pivot(const DFront* d_fronts, int32_t n_fronts, const double* d_fstore, double* out_min,
              int64_t* out_pos, void* stream);
int launch_factor_dag(const FactorArgs& A, int grid, void* stream);

std::string& last_error();

// number of kernel launches issued by this library (gpu_launches evidence for bench.py)
void count_launch(int64_t n = 1);
int64_t launch_count();

int launch_shell(bool derivs, int32_t elem_type, int64_t n_elems, int32_t batch, const int32_t* conn,
                 const double* pos, const double* rest, int64_t vstride, const double* params,
                 int64_t pstride, double* out1, double* out2, int64_t bstride, void* stream,
                 int rest_comp_mask = 7);

// returns 0 ok, 1 singular (pivot_index set), 5 invalid
int build_symbolic(Symbolic& s, const SymOptions& opt, int64_t* pivot_index);

}  // namespace sgn
