// Persistent dependency-driven multifrontal LDL^T factorization on B200 (sm_100a).
//
// Replaces, on the GPU, the reference's SuperLU numeric LU of the stabilized KKT
// (reference pkg/src/sgnopt/linear_solvers.py:87 + :111-127) -- see numeric.cu for the
// surrounding C ABI.  ONE launch per factorization: resident CTAs take tasks in the
// topological order built by symbolic.cpp ("persistent factorization tasks") from a
// global head counter, wait on per-tile / per-step / per-front counters derived from the
// task coordinates (gpu-scope acquire loads), run the task and release its counters.
//
//   F_ASM    one 32x32 tile of a front: original KKT entries, the signed stabilization
//            shift, then the children's update matrices extend-added in child order
//            (atomic free, bitwise deterministic).
//   F_PANEL  one pivot step of a front: LDL^T of the 32x32 diagonal block (2x2 pivots on
//            matched (x_i, lambda_j) pairs or 1x1), then TRSM of up to four 32-row tiles
//            below it: W = P L11^{-T} (kept transposed in the front's unused upper
//            triangle) and L21 = W D^{-1}.
//   F_UPDATE one 32x32 Schur tile C -= L21_i W_j^T on the FP64 tensor pipe (DMMA).
//   F_ZPANEL one 32-row slab of the solve panel Z = [I; L21] L11^{-1}.
//
// Every value produced inside the launch is read with ld.global.cg (L2): a persistent
// CTA keeps its L1 across tasks and must never see a stale line.  Bodies are compact
// loops (the whole kernel shares one instruction cache).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <string>

#include "../../include/sgn_b200.h"
#include "sgn_internal.h"

namespace {

using sgn::DFront;
using sgn::kTile;

constexpr int kFThreads = 128;

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_ge(const int* p, int target) {
  while (ld_acq(p) < target) __nanosleep(20);
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {     // global -> shared, 16 B, L2 only
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// Shared memory (dynamic, ~53 KB): five raw 32 x 40 tiles, each viewed either row-major
// with stride 33 (one row per lane: conflict-free) or K-major with stride 40 (DMMA
// fragment reads (row g, k q) and the coalesced staging stores both conflict-free).
constexpr int kTileWords = kTile * 40;
typedef double (*V33)[kTile + 1];
typedef double (*V40)[40];
struct Smem {
  double a[kTileWords];
  double b[4][kTileWords];
  double2 colbuf[2 * kTile];        // panel: pivot columns broadcast
  double dinv[kTile][3];            // per pivot block: (ia, ib, ic) or (1/d)
  unsigned long long* tr;           // this task's trace words (diagnostics) or null
  int bad;
};
__device__ __forceinline__ V33 v33(double* p) { return reinterpret_cast<V33>(p); }
__device__ __forceinline__ V40 v40(double* p) { return reinterpret_cast<V40>(p); }

__device__ __forceinline__ void tmark(Smem& S, int slot) {
  if (threadIdx.x == 0 && S.tr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    S.tr[slot] = t;
  }
}

__device__ __forceinline__ double* front_ptr(const sgn::FactorArgs& A, const DFront& F, int b) {
  return A.fstore + (int64_t)b * A.fstride + F.foff;
}

// ---------------------------------------------------------------------------------------
__device__ void f_asm(const sgn::FactorArgs& A, const DFront& F, int b, int ti, int tj, Smem& S) {
  double (*tile)[kTile + 1] = v33(S.a);
  const int tid = threadIdx.x;
  for (int e = tid; e < kTile * kTile; e += kFThreads) tile[e >> 5][e & 31] = 0.0;
  __syncthreads();
  const double* vals = A.values + (int64_t)b * A.vstride;
  {
    const int64_t tg = F.tile_base + (int64_t)ti * (ti + 1) / 2 + tj;
    const int64_t e0 = A.tile_ptr[tg], e1 = A.tile_ptr[tg + 1];
    for (int64_t e = e0 + tid; e < e1; e += kFThreads) {
      const int loc = A.tile_loc[e];
      tile[loc >> 5][loc & 31] = vals[A.tile_nnz[e]];
    }
  }
  __syncthreads();
  const int i0 = sgn::tile_lo(F.npiv, ti), i1 = sgn::tile_hi(F.npiv, F.nrow, ti);
  const int j0 = sgn::tile_lo(F.npiv, tj), j1 = sgn::tile_hi(F.npiv, F.nrow, tj);
  if (ti == tj && i0 < F.npiv && tid < i1 - i0) {
    const int8_t kd = A.kind_pos[F.first + i0 + tid];
    if (kd == 1) tile[tid][tid] += A.eps_xv ? A.eps_xv[b] : A.eps_x;
    else if (kd == 2) tile[tid][tid] -= A.eps_lv ? A.eps_lv[b] : A.eps_l;
  }
  const double* fb = A.fstore + (int64_t)b * A.fstride;
  for (int ci = F.child_begin; ci < F.child_end; ++ci) {
    const DFront C = A.fronts[A.children[ci]];
    const int cn = C.nrow - C.npiv;
    __syncthreads();
    if (cn == 0) continue;
    const int32_t* rc = A.rel + C.rel_off;
    const int32_t* rt = A.reltile + C.woff;
    const int r_lo = rt[ti], r_hi = rt[ti + 1], s_lo = rt[tj], s_hi = rt[tj + 1];
    const int nr = r_hi - r_lo, ns = s_hi - s_lo;
    if (nr <= 0 || ns <= 0) continue;
    const double* U = fb + C.foff;
    const int64_t ldc = sgn::front_ld(C.nrow);
    for (int idx = tid; idx < nr * ns; idx += kFThreads) {
      const int r = r_lo + idx % nr, s = s_lo + idx / nr;
      if (r >= s) tile[rc[r] - i0][rc[s] - j0] += __ldcg(U + (int64_t)(C.npiv + s) * ldc + C.npiv + r);
    }
  }
  __syncthreads();
  double* Fm = front_ptr(A, F, b);
  const int64_t ld = sgn::front_ld(F.nrow);
  for (int e = tid; e < kTile * kTile; e += kFThreads) {
    const int ii = e & 31, jj = e >> 5;
    const int gi = i0 + ii, gj = j0 + jj;
    if (gi < i1 && gj < j1) Fm[(int64_t)gj * ld + gi] = tile[ii][jj];
  }
  if (ti == 0 && tj == 0 && F.npiv > 0)     // D_0 is factored by the caller (single site)
    for (int e = tid; e < kTile * kTile; e += kFThreads)
      if ((e >> 5) < (e & 31)) tile[e >> 5][e & 31] = 0.0;
}

// F_ASM with k = 1: the 64x64 block of tiles {ti, ti+1} x {tj, tj+1} in one task (the
// lower tiles of it; ti, tj even).  Same sources and order as f_asm per entry: original
// entries, the signed shift on pivot diagonals, then every child's update block extend-
// added in child order (bitwise identical to four f_asm tiles), with one pass of the
// latency chain (tile lists, child fronts, relative rows) for up to four tiles.  Block
// buffer: 64 x 65 doubles in S.b (row-major, conflict-free column write-out); a block
// holding tile (0, 0) also leaves that tile in S.a for the caller's D_0 factorization.
constexpr int kA2 = 65;
__device__ void f_asm2(const sgn::FactorArgs& A, const DFront& F, int b, int ti, int tj, Smem& S) {
  static_assert(64 * kA2 <= 4 * kTileWords, "64x64 assembly block fits S.b");
  double* Bk = &S.b[0][0];
  const int tid = threadIdx.x;
  const int T = sgn::ntiles_front(F.npiv, F.nrow);
  // children's metadata (front, relative-row ranges of this block), one child per thread, into
  // S.a while the block is cleared and the original entries load: the per-child chain
  // children[] -> fronts[] -> reltile[] is paid once, in parallel, not once per child in turn
  struct AsmChild { const double* Ur; const int32_t* rc; int64_t ldc; int r_lo, r_hi, s_lo, s_hi; };
  constexpr int kMaxMeta = (int)(kTileWords * sizeof(double) / sizeof(AsmChild));
  AsmChild* cm = reinterpret_cast<AsmChild*>(S.a);
  const int nch = F.child_end - F.child_begin;
  const double* fb = A.fstore + (int64_t)b * A.fstride;
  for (int c = tid; c < min(nch, kMaxMeta); c += kFThreads) {
    const DFront C = A.fronts[A.children[F.child_begin + c]];
    AsmChild m;
    m.Ur = nullptr; m.rc = nullptr; m.ldc = 0; m.r_lo = m.r_hi = m.s_lo = m.s_hi = 0;
    if (C.nrow > C.npiv) {
      const int32_t* rt = A.reltile + C.woff;
      m.r_lo = rt[ti]; m.r_hi = rt[min(ti + 2, T)]; m.s_lo = rt[tj]; m.s_hi = rt[min(tj + 2, T)];
      m.rc = A.rel + C.rel_off;
      m.ldc = sgn::front_ld(C.nrow);
      m.Ur = fb + C.foff + (int64_t)C.npiv * m.ldc + C.npiv;
    }
    cm[c] = m;
  }
  for (int e = tid; e < 64 * kA2; e += kFThreads) Bk[e] = 0.0;
  __syncthreads();
  const double* vals = A.values + (int64_t)b * A.vstride;
  const int xlo_i = sgn::tile_lo(F.npiv, ti), xlo_j = sgn::tile_lo(F.npiv, tj);
  const int mid_i = (ti + 1 < T) ? sgn::tile_lo(F.npiv, ti + 1) : (1 << 30);
  const int mid_j = (tj + 1 < T) ? sgn::tile_lo(F.npiv, tj + 1) : (1 << 30);
  // front-local row / col -> block index (the second tile starts at 32)
  auto bi = [&](int g) { return g < mid_i ? g - xlo_i : 32 + g - mid_i; };
  auto bj = [&](int g) { return g < mid_j ? g - xlo_j : 32 + g - mid_j; };
  for (int x = ti; x < min(ti + 2, T); ++x)
    for (int y = tj; y < min(tj + 2, T); ++y) {
      if (x < y) continue;
      const int64_t tg = F.tile_base + (int64_t)x * (x + 1) / 2 + y;
      const int64_t e0 = A.tile_ptr[tg], e1 = A.tile_ptr[tg + 1];
      const int ro = 32 * (x - ti), co = 32 * (y - tj);
      for (int64_t e = e0 + tid; e < e1; e += kFThreads) {
        const int loc = A.tile_loc[e];
        Bk[(ro + (loc >> 5)) * kA2 + co + (loc & 31)] = vals[A.tile_nnz[e]];
      }
    }
  __syncthreads();
  if (ti == tj) {                               // signed shift on the pivot diagonals
    const int d = tid & 63, x = ti + (d >> 5);
    if (tid < 64 && x < T) {
      const int gi = sgn::tile_lo(F.npiv, x) + (d & 31);
      if (gi < min(F.npiv, sgn::tile_hi(F.npiv, F.nrow, x))) {
        const int8_t kd = A.kind_pos[F.first + gi];
        if (kd == 1) Bk[d * kA2 + d] += A.eps_xv ? A.eps_xv[b] : A.eps_x;
        else if (kd == 2) Bk[d * kA2 + d] -= A.eps_lv ? A.eps_lv[b] : A.eps_l;
      }
    }
  }
  __syncthreads();                              // original entries and the shift are in place
  bool dirty = false;                           // adds of a child in flight since the last barrier
  for (int ci = 0; ci < nch; ++ci) {
    AsmChild m;
    if (ci < kMaxMeta) {
      m = cm[ci];
    } else {                                    // (more children than metadata slots: direct loads)
      const DFront C = A.fronts[A.children[F.child_begin + ci]];
      m.Ur = nullptr; m.rc = nullptr; m.ldc = 0; m.r_lo = m.r_hi = m.s_lo = m.s_hi = 0;
      if (C.nrow > C.npiv) {
        const int32_t* rt = A.reltile + C.woff;
        m.r_lo = rt[ti]; m.r_hi = rt[min(ti + 2, T)]; m.s_lo = rt[tj]; m.s_hi = rt[min(tj + 2, T)];
        m.rc = A.rel + C.rel_off;
        m.ldc = sgn::front_ld(C.nrow);
        m.Ur = fb + C.foff + (int64_t)C.npiv * m.ldc + C.npiv;
      }
    }
    const int32_t* rc = m.rc;
    const int r_lo = m.r_lo, r_hi = m.r_hi, s_lo = m.s_lo, s_hi = m.s_hi;
    const int nr = r_hi - r_lo, ns = s_hi - s_lo;
    if (nr <= 0 || ns <= 0) continue;           // (uniform: the metadata is the same for every thread)
    if (dirty) __syncthreads();                 // children are added one after another, in child order
    dirty = true;
    const int64_t ldc = m.ldc;
    // A warp per child column, a lane per child row (nr <= 64: two rows per lane, their block
    // rows looked up once per child); four columns = 8 entries per thread in flight: the loads
    // (child update block, coalesced along the column) first, then the shared-memory adds
    // (every entry of one child lands on its own position)
    const int lane = tid & 31, warp = tid >> 5;
    const int ra = r_lo + lane, rb = ra + 32;
    const int ba = (ra < r_hi) ? bi(rc[ra]) * kA2 : -1;
    const int bb = (rb < r_hi) ? bi(rc[rb]) * kA2 : -1;
    const double* Ur = m.Ur;
    // the warp's <= 16 columns (warp + 4 i): their block columns are loaded by lanes i next to
    // the row lookups above (one latency) and handed out by shuffles
    const int myc = warp + 4 * (lane & 15);
    const int cjl = (myc < ns) ? bj(rc[s_lo + myc]) : 0;
    for (int sb = warp, pass = 0; sb < ns; sb += 16, ++pass) {
      double u[8];
      int di[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int so = sb + 4 * q, s = s_lo + so;
        const int cj = __shfl_sync(0xffffffffu, cjl, 4 * pass + q);
        di[2 * q] = di[2 * q + 1] = -1;
        u[2 * q] = u[2 * q + 1] = 0.0;
        if (so < ns) {
          const double* col = Ur + (int64_t)s * ldc;
          if (ba >= 0 && ra >= s) { u[2 * q] = __ldcg(col + ra); di[2 * q] = ba + cj; }
          if (bb >= 0 && rb >= s) { u[2 * q + 1] = __ldcg(col + rb); di[2 * q + 1] = bb + cj; }
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (di[q] >= 0) Bk[di[q]] += u[q];
    }
  }
  __syncthreads();
  double* Fm = front_ptr(A, F, b);
  const int64_t ld = sgn::front_ld(F.nrow);
  {   // write-out: this thread's block row is fixed (kFThreads = 2 x 64), columns tid >> 6, +2, ...
    const int ii = tid & 63, x = ti + (ii >> 5);
    const int gi = (x < T) ? sgn::tile_lo(F.npiv, x) + (ii & 31) : 0;
    const bool rok = x < T && gi < sgn::tile_hi(F.npiv, F.nrow, x);
    for (int yh = 0; yh < 2; ++yh) {
      const int y = tj + yh;
      if (!rok || y >= T || x < y) continue;
      const int lo = sgn::tile_lo(F.npiv, y), hi = sgn::tile_hi(F.npiv, F.nrow, y);
      double* col = Fm + (int64_t)lo * ld + gi;
      const double* brow_ = Bk + ii * kA2 + 32 * yh;
#pragma unroll 4
      for (int jl = tid >> 6; jl < 32; jl += 2)
        if (lo + jl < hi) col[(int64_t)jl * ld] = brow_[jl];
    }
  }
  if (ti == 0 && tj == 0 && F.npiv > 0) {       // D_0 for the caller: tile (0, 0), lower part
    double (*tile)[kTile + 1] = v33(S.a);
    for (int e = tid; e < kTile * kTile; e += kFThreads) {
      const int r = e >> 5, c = e & 31;
      tile[r][c] = (r >= c) ? Bk[r * kA2 + c] : 0.0;
    }
  }
}

// LDL^T of the w x w diagonal block by one warp (lane i = row i), rows in registers,
// fully unrolled so every register index is static; the two pivot columns of each step
// are broadcast through smem (colbuf) -- measured 2.2x faster than shuffles and 9x faster
// than a runtime-loop register window (profiles/micro/diag_factor_bench.cu).  The factored
// values (L below the pivot blocks, D on them) are written back into D.  Returns the
// first zero / non-finite pivot position or 1 << 30.
template <int PT>
__device__ int factor_diag(double (*D)[kTile + 1], double2* colbuf, int w) {
  const int i = threadIdx.x & 31;
  int first_bad = 1 << 30;
  double d[kTile];
#pragma unroll
  for (int k = 0; k < kTile; ++k) d[k] = (k <= i) ? D[i][k] : 0.0;
#pragma unroll
  for (int j = 0; j < kTile; j += PT) {
    const bool act = (j < w);
    colbuf[i] = make_double2(d[j], PT == 2 ? d[j + 1] : 0.0);
    __syncwarp();
    if (PT == 2) {
      const double2 pj = colbuf[j], pj1 = colbuf[j + 1];
      const double a = pj.x, bb = pj1.x, c = pj1.y;
      double det = a * c - bb * bb;
      first_bad = (act && (det == 0.0 || !isfinite(det)) && first_bad > j) ? j : first_bad;
      det = (act && det != 0.0 && isfinite(det)) ? det : 1.0;
      const double rdet = 1.0 / det;
      const double ia = c * rdet, ib = -bb * rdet, ic = a * rdet;
      const bool below = act && (i > j + 1) && (i < w);
      const double x0 = d[j], x1 = d[j + 1];
      const double l0 = below ? x0 * ia + x1 * ib : 0.0;
      const double l1 = below ? x0 * ib + x1 * ic : 0.0;
#pragma unroll
      for (int k = j + 2; k < kTile; ++k) {
        const double2 y = colbuf[k];
        d[k] = fma(-l1, y.y, fma(-l0, y.x, d[k]));   // right of the diagonal: junk, never read
      }
      d[j] = below ? l0 : d[j];
      d[j + 1] = below ? l1 : d[j + 1];
    } else {
      double dj = colbuf[j].x;
      first_bad = (act && (dj == 0.0 || !isfinite(dj)) && first_bad > j) ? j : first_bad;
      dj = (act && dj != 0.0 && isfinite(dj)) ? dj : 1.0;
      const bool below = act && (i > j) && (i < w);
      const double l = below ? d[j] * (1.0 / dj) : 0.0;
#pragma unroll
      for (int k = j + 1; k < kTile; ++k) d[k] = fma(-l, colbuf[k].x, d[k]);
      d[j] = below ? l : d[j];
    }
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < kTile; ++k) if (k <= i) D[i][k] = d[k];
  return first_bad;
}

// W = P L11^{-T} for one 32-row tile (lane = row), right-looking, row in registers, fully
// unrolled; Lt[cp][c] = L11[c][cp] (unit lower, D slots cleared) broadcast from smem.
__device__ __forceinline__ void trsm_rows(double (*Pw)[kTile + 1], const double (*Lt)[kTile + 1]) {
  const int lane = threadIdx.x & 31;
  double p[kTile];
#pragma unroll
  for (int m = 0; m < kTile; ++m) p[m] = Pw[lane][m];
#pragma unroll
  for (int cp = 0; cp < kTile; ++cp) {
    const double pc = p[cp];
#pragma unroll
    for (int c = cp + 1; c < kTile; ++c) p[c] = fma(-pc, Lt[cp][c], p[c]);
  }
#pragma unroll
  for (int m = 0; m < kTile; ++m) Pw[lane][m] = p[m];
}

// Factor the w x w pivot block of step k held (lower part) in smem tile D and publish it
// to the step's scratch [D | L^T | D^-1]: the factored block (Z-panel / solve), the unit
// lower L^T with the 2x2 D slots cleared (TRSM, Z panel) and the pivot-block inverses.
// Records the first bad pivot in status.  All threads of the CTA take part.
__device__ __forceinline__ void factor_publish(const sgn::FactorArgs& A, const DFront& F, int b, int k,
                                            double (*D)[kTile + 1], Smem& S) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int j0 = k * kTile, w = min(kTile, F.npiv - j0);
  __syncthreads();
  if (warp == 0) {
    const int bad = (F.pivtype == 2) ? factor_diag<2>(D, S.colbuf, w) : factor_diag<1>(D, S.colbuf, w);
    if (lane == 0 && bad < (1 << 30)) atomicMin(&A.status[b], (long long)A.perm[F.first + j0 + bad]);
  }
  __syncthreads();
  tmark(S, 6);
  double* ds = A.dscr + (int64_t)b * A.dstride + F.doff + (int64_t)k * sgn::kDiagStride;
  for (int e = tid; e < kTile * kTile; e += kFThreads) {
    const int r = e >> 5, c = e & 31;
    ds[e] = D[r][c];
    const int cp = r, cc = c;                                 // L^T[cp][cc] = L[cc][cp]
    const bool dslot = F.pivtype == 2 && (cp & 1) == 0 && cc == cp + 1;
    ds[kTile * kTile + e] = (cc > cp && cc < w && !dslot) ? D[cc][cp] : 0.0;
  }
  if (tid < w) {
    double* di = ds + 2 * kTile * kTile + 3 * tid;
    if (F.pivtype == 2) {
      const int t0 = tid & ~1;
      const double a = D[t0][t0], bb = D[t0 + 1][t0], cc = D[t0 + 1][t0 + 1];
      const double rdet = 1.0 / (a * cc - bb * bb);
      di[0] = cc * rdet; di[1] = -bb * rdet; di[2] = a * rdet;
    } else {
      di[0] = 1.0 / D[tid][tid]; di[1] = 0.0; di[2] = 0.0;
    }
  }
}

// TRSM of step k for row tile k+1 (t = 0, warp 0) or tiles k+2+4(t-1).. (t >= 1, a warp
// each): W = P L11^{-T} (kept transposed in the front's upper triangle) and L21 = W D^-1,
// with L11^T and D^-1 read from the step's scratch (factored once by its producer).
__device__ int f_panel_pre(const sgn::FactorArgs& A, const DFront& F, int b, int k, int t, Smem& S) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* Fm = front_ptr(A, F, b);
  const int64_t ld = sgn::front_ld(F.nrow);
  const int j0 = k * kTile, w = min(kTile, F.npiv - j0);
  const int T = sgn::ntiles_front(F.npiv, F.nrow);
  double (*Lt)[kTile + 1] = v33(S.a);
  const int ti = (t == 0) ? (warp == 0 ? k + 1 : T) : k + 2 + 4 * (t - 1) + warp;
  const int lo = (ti < T) ? sgn::tile_lo(F.npiv, ti) : 0;
  const int nr = (ti < T) ? sgn::tile_hi(F.npiv, F.nrow, ti) - lo : 0;
  double (*Pw)[kTile + 1] = v33(S.b[warp]);
  // the row tiles are final (waited by the caller): load them while D_k may still be in
  // production, then wait for D_k and read its published L^T / D^-1
  if (nr > 0) {
    double v[kTile];
#pragma unroll
    for (int j = 0; j < kTile; ++j) v[j] = (lane < nr && j < w) ? __ldcg(Fm + (int64_t)(j0 + j) * ld + lo + lane) : 0.0;
#pragma unroll
    for (int j = 0; j < kTile; ++j) Pw[lane][j] = v[j];
  }
  if (tid == 0) {
    const int P = sgn::ptiles(F.npiv);
    spin_ge(A.cnt + (int64_t)b * A.n_fcnt + F.cbase + sgn::cnt_diag(P, k), 1);
  }
  __syncthreads();
  const double* ds = A.dscr + (int64_t)b * A.dstride + F.doff + (int64_t)k * sgn::kDiagStride;
  for (int e = tid; e < kTile * kTile; e += kFThreads) Lt[e >> 5][e & 31] = __ldcg(ds + kTile * kTile + e);
  if (tid < 3 * kTile) (&S.dinv[0][0])[tid] = __ldcg(ds + 2 * kTile * kTile + tid);
  return nr;
}

// after the substitution: W -> the front's upper triangle (transposed), L21 = W D^-1
__device__ void f_panel_post(const sgn::FactorArgs& A, const DFront& F, int b, int k, int t, int nr, Smem& S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (nr == 0) return;
  double* Fm = front_ptr(A, F, b);
  const int64_t ld = sgn::front_ld(F.nrow);
  const int j0 = k * kTile, w = min(kTile, F.npiv - j0);
  const int ti = (t == 0) ? k + 1 : k + 2 + 4 * (t - 1) + warp;
  const int lo = sgn::tile_lo(F.npiv, ti);
  double (*Pw)[kTile + 1] = v33(S.b[warp]);
  for (int r = 0; r < nr; ++r)
    if (lane < w) Fm[(int64_t)(lo + r) * ld + j0 + lane] = Pw[r][lane];
  if (lane < nr) {
    for (int c = 0; c < w; ++c) {
      double l;
      if (F.pivtype == 2) {
        const int c0 = c & ~1;
        const double x0 = Pw[lane][c0], x1 = Pw[lane][c0 + 1];
        l = (c == c0) ? x0 * S.dinv[c0][0] + x1 * S.dinv[c0][1] : x0 * S.dinv[c0][1] + x1 * S.dinv[c0][2];
      } else {
        l = Pw[lane][c] * S.dinv[c][0];
      }
      Fm[(int64_t)(j0 + c) * ld + lo + lane] = l;
    }
  }
}

// C[ti, tj] -= L21[ti, step k] W[tj, step k]^T   (mma.sync.m8n8k4.f64 -> DMMA).
// diag: the last update of pivot tile (k+1, k+1) -- the result stays in smem (S.b[1]) and
// is factored and published as D_{k+1} instead of being written back.
__device__ void f_update(const sgn::FactorArgs& A, const DFront& F, int b, int k0, int k, int ti, int tj, Smem& S,
                         bool diag = false) {
  V40 Ak = v40(S.a);          // Ak[c][i] = L21[lo_i + i, j0 + c]
  V40 Bk = v40(S.b[0]);       // Bk[c][j] = W[lo_j + j, j0 + c]
  const int tid = threadIdx.x;
  double* Fm = front_ptr(A, F, b);
  const int64_t ld = sgn::front_ld(F.nrow);
  const int lo_i = sgn::tile_lo(F.npiv, ti), nr = sgn::tile_hi(F.npiv, F.nrow, ti) - lo_i;
  const int lo_j = sgn::tile_lo(F.npiv, tj), nc = sgn::tile_hi(F.npiv, F.nrow, tj) - lo_j;
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int row0 = warp * 8;
  const int i = row0 + g;
  double va[8], vb[8];
  V40 Cs = v40(S.b[2]);       // Cs[j][i] = C(lo_i + i, lo_j + j): staged, not held in registers
  // C is final up to step k0-1 (waited by the caller): load it while step k's panels may
  // still be running, then wait for them and stream the L21 / W tiles of steps k0..k
  {
    double cv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * kFThreads;
      const int r = e & 31, c = e >> 5;
      cv[u] = (r < nr && c < nc && (ti != tj || r >= c)) ? __ldcg(Fm + (int64_t)(lo_j + c) * ld + lo_i + r) : 0.0;
    }
    if (tid == 0) {
      // the TRSM tasks of step k that wrote row tiles ti and tj (the diagonal update: k+1)
      const int* cfb = A.cnt + (int64_t)b * A.n_fcnt + F.cbase;
      spin_ge(cfb + sgn::cnt_pant(F.npiv, F.nrow, k, sgn::pan_task_of(k, ti)), 1);
      if (tj != ti) spin_ge(cfb + sgn::cnt_pant(F.npiv, F.nrow, k, sgn::pan_task_of(k, tj)), 1);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * kFThreads;
      Cs[e >> 5][e & 31] = cv[u];
    }
  }
  __syncthreads();
#define SGN_LOAD_STEP(S_)                                                                          \
  do {                                                                                             \
    const int j0_ = (S_) * kTile, w_ = min(kTile, F.npiv - j0_);                                   \
    _Pragma("unroll") for (int u = 0; u < 8; ++u) {                                                \
      const int e = tid + u * kFThreads;                                                           \
      const int r = e & 31, c = e >> 5;                                                            \
      va[u] = (r < nr && c < w_) ? __ldcg(Fm + (int64_t)(j0_ + c) * ld + lo_i + r) : 0.0;          \
      vb[u] = (c < nc && r < w_) ? __ldcg(Fm + (int64_t)(lo_j + c) * ld + j0_ + r) : 0.0;          \
    }                                                                                              \
  } while (0)
  SGN_LOAD_STEP(k0);   // 16 operand loads in flight together
  double acc[4][2];
#pragma unroll
  for (int nf = 0; nf < 4; ++nf) acc[nf][0] = acc[nf][1] = 0.0;
  for (int s = k0; s <= k; ++s) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * kFThreads;
      const int r = e & 31, c = e >> 5;
      Ak[c][r] = va[u];
      Bk[r][c] = vb[u];
    }
    __syncthreads();
    if (s < k) SGN_LOAD_STEP(s + 1);      // next step's operands in flight during the DMMAs
    tmark(S, 4);
#pragma unroll
    for (int kk = 0; kk < kTile; kk += 4) {
      const double a = Ak[kk + q][row0 + g];
#pragma unroll
      for (int nf = 0; nf < 4; ++nf) dmma_8x8x4(acc[nf][0], acc[nf][1], a, Bk[kk + q][nf * 8 + g]);
    }
    __syncthreads();
  }
  tmark(S, 5);
  if (diag) {
    double (*Dn)[kTile + 1] = v33(S.b[1]);
#pragma unroll
    for (int nf = 0; nf < 4; ++nf)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = nf * 8 + 2 * q + h;
        Dn[i][j] = (i < nr && j < nc && i >= j) ? Cs[j][i] - acc[nf][h] : 0.0;
      }
    return;   // the caller factors and publishes D_{k+1}
  }
  if (i < nr) {
#pragma unroll
    for (int nf = 0; nf < 4; ++nf)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = nf * 8 + 2 * q + h;
        if (j < nc && (ti != tj || i >= j)) Fm[(int64_t)(lo_j + j) * ld + lo_i + i] = Cs[j][i] - acc[nf][h];
      }
  }
}

// 64x64 DMMA block products of the factorization (each warp owns a 32x32 quarter as 4x4
// m8n8k4 fragments, acc in registers, so a streamed 32-wide step (A 64x32, B 64x32) feeds
// twice the DMMA work per operand byte of the 32x32 bodies; profiles/micro/upd_bench.cu:
// 26.5 vs 12.9 TFLOP/s).  Smem: A K-major (stride 68), B N-major (stride 36): fragment
// reads and staging stores are conflict-free.
//   ZP = false, F_UPD2: C(ti..ti+1, tj..tj+1) -= sum_{s=k0..k} L21(rows, step s) W(cols, step s)^T;
//                tiles past the front, and the upper tile (ti, tj+1) of a diagonal block,
//                are neither read nor written.
//   ZP = true,  F_ZPAN2: Z(t..t+1, cb..cb+1) = sum_{j=cb}^{P-1} L(t..t+1, j) Z(j, cb..cb+1) for
//                struct tiles t >= P (Z(cb, cb+1) = 0, so both columns sum from j = cb).
constexpr int kU2A = 68, kU2B = 36;
#ifndef SGN_UPD_RED
#define SGN_UPD_RED 1
#endif
constexpr bool kUpdRed = SGN_UPD_RED != 0;   // C -= acc by red.global.add.f64 (1) or load / subtract / store (0)
// NB = 32: one column tile (the row-paired single-column updates: look-ahead and single-step
// columns, unpaired groups); warps own 32x16 quarters (4x2 fragments).
template <bool ZP, int NB>
__device__ void f_block64(const sgn::FactorArgs& A, const DFront& F, int b, int k0, int k, int ti, int tj, Smem& S) {
  static_assert(NB == 64 || NB == 32, "block width");
  constexpr int NF = NB / 16;             // n fragments per warp
  static_assert(32 * kU2A + 64 * kU2B <= 5 * kTileWords, "64x64 operands fit the tile buffers");
  double* As = reinterpret_cast<double*>(&S);   // [32][kU2A] As[c][r] = L(row(r), j0 + c)  (S.a, S.b)
  double* Bs = As + 32 * kU2A;                  // [64][kU2B] Bs[j][c] = W(col(j), j0 + c) | Z(j0 + c, col j)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * (NB / 2);
  double* Fm = front_ptr(A, F, b);
  double* Zm = A.zstore + (int64_t)b * A.zstride + F.zoff;
  const int64_t ld = sgn::front_ld(F.nrow);
  const int T = sgn::ntiles_front(F.npiv, F.nrow);
  // row r of the block -> front row (or -1): tile t0 + (r >> 5), row r & 31 of that tile
  auto brow = [&](int t0, int r) -> int {
    const int t = t0 + (r >> 5);
    if (t >= T) return -1;
    const int lo = sgn::tile_lo(F.npiv, t);
    return (lo + (r & 31) < sgn::tile_hi(F.npiv, F.nrow, t)) ? lo + (r & 31) : -1;
  };
  // column j of the block -> W row (update) or Z column (Z panel), or -1
  auto bcol = [&](int j) -> int {
    if (!ZP) return brow(tj, j);
    const int c = 32 * tj + j;
    return c < F.npiv ? c : -1;
  };
  const int ra = brow(ti, tid & 63);      // this thread's A staging row (fixed)
  double acc[4][NF][2];
#pragma unroll
  for (int mf = 0; mf < 4; ++mf)
#pragma unroll
    for (int nf = 0; nf < NF; ++nf) acc[mf][nf][0] = acc[mf][nf][1] = 0.0;
  // one 32-wide step through registers (partial steps, Z's structurally-zero upper block,
  // fronts with an odd npiv)
  auto step_reg = [&](int s) {
    const int j0 = s * kTile, w = min(kTile, F.npiv - j0);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = (tid >> 6) + 2 * (u + 8 * hh);
        v[u] = (ra >= 0 && c < w) ? __ldcg(Fm + (int64_t)(j0 + c) * ld + ra) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) As[((tid >> 6) + 2 * (u + 8 * hh)) * kU2A + (tid & 63)] = v[u];
    }
#pragma unroll
    for (int hh = 0; hh < NB / 32; ++hh) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = (tid >> 5) + 4 * (u + 8 * hh), cb = bcol(j);
        const double* src = ZP ? Zm : Fm;
        // Z(j0 + lane, col) of a pivot tile above the column's block is structurally zero
        // and never stored (only the first column block's s = tj step reaches it)
        const bool zup = ZP && s < tj + (j >> 5);
        v[u] = (cb >= 0 && lane < w && !zup) ? __ldcg(src + (int64_t)cb * ld + j0 + lane) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) Bs[((tid >> 5) + 4 * (u + 8 * hh)) * kU2B + lane] = v[u];
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTile; kk += 4) {
      double fa[4], fb[NF];
#pragma unroll
      for (int mf = 0; mf < 4; ++mf) fa[mf] = As[(kk + q) * kU2A + wm + 8 * mf + g];
#pragma unroll
      for (int nf = 0; nf < NF; ++nf) fb[nf] = Bs[(wn + 8 * nf + g) * kU2B + kk + q];
#pragma unroll
      for (int mf = 0; mf < 4; ++mf)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], fa[mf], fb[nf]);
    }
    __syncthreads();
  };
  // full 32-wide steps with 16-byte aligned operands (even npiv: every tile starts at an even
  // row; ld is even) stream through a cp.async.cg double buffer of 16-wide half steps, so the
  // next half step's operands are in flight during the DMMAs (profiles/micro/upd_bench.cu:
  // v64a 30.3 vs v64 26.5 TFLOP/s).  Rows / columns past the block read a clamped valid
  // address: their products only reach accumulators that are never stored.
  const int sa = ZP ? k0 + 1 : k0;
  const int sb = (F.npiv & 1) ? sa - 1 : min(k, (F.npiv >> 5) - 1);
  if (ZP) step_reg(k0);
  if (sb >= sa) {
    double* As2 = As;                           // [2][16][kU2A]
    double* Bs2 = As + 2 * 16 * kU2A;           // [2][NB][kA2B]
    constexpr int kA2B = 20;
    static_assert(2 * 16 * kU2A + 2 * 64 * kA2B <= 5 * kTileWords, "cp.async buffers fit");
    const double* bsrc = ZP ? Zm : Fm;
    // this thread's staging addresses are fixed for the task (kFThreads is a multiple of 32 and
    // of 8): the A row pair and the NB / 16 B rows are resolved once, not per half step
    const int cha = tid & 31, chb = tid & 7;
    const int gra = max(brow(ti, 2 * cha), 0);
    const double* asrc = Fm + gra;
    const double* bsrcu[NB / 16];
#pragma unroll
    for (int u = 0; u < NB / 16; ++u) bsrcu[u] = bsrc + (int64_t)max(bcol((tid >> 3) + 16 * u), 0) * ld + 2 * chb;
    auto issue = [&](int hs, int buf) {
      const int c0 = (sa + (hs >> 1)) * kTile + 16 * (hs & 1);
#pragma unroll
      for (int u = 0; u < 4; ++u) {             // A: 16 columns x 32 row pairs
        const int c = (tid >> 5) + 4 * u;
        cp16(&As2[(buf * 16 + c) * kU2A + 2 * cha], asrc + (int64_t)(c0 + c) * ld);
      }
#pragma unroll
      for (int u = 0; u < NB / 16; ++u) {       // B: NB rows x 8 k pairs
        const int j = (tid >> 3) + 16 * u;
        cp16(&Bs2[(buf * 64 + j) * kA2B + 2 * chb], bsrcu[u] + c0);
      }
      cp_commit();
    };
    const int nh = 2 * (sb - sa + 1);
    issue(0, 0);
    for (int hs = 0; hs < nh; ++hs) {
      const int buf = hs & 1;
      if (hs + 1 < nh) { issue(hs + 1, buf ^ 1); cp_wait<1>(); } else { cp_wait<0>(); }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 16; kk += 4) {
        double fa[4], fb[NF];
#pragma unroll
        for (int mf = 0; mf < 4; ++mf) fa[mf] = As2[(buf * 16 + kk + q) * kU2A + wm + 8 * mf + g];
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) fb[nf] = Bs2[(buf * 64 + wn + 8 * nf + g) * kA2B + kk + q];
#pragma unroll
        for (int mf = 0; mf < 4; ++mf)
#pragma unroll
          for (int nf = 0; nf < NF; ++nf) dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], fa[mf], fb[nf]);
      }
      __syncthreads();
    }
  }
  for (int s = max(sa, sb + 1); s <= k; ++s) step_reg(s);
  // C -= acc: the C loads of one fragment row (2 NF values per thread) are issued together,
  // then subtracted and stored -- a load / store pair per value would serialize one memory
  // latency per value behind the possibly-aliasing store before it (ncu: 19 % of the
  // config-4 factorization's stall samples sat on that line)
  int gcn[NF][2];
#pragma unroll
  for (int nf = 0; nf < NF; ++nf)
#pragma unroll
    for (int h = 0; h < 2; ++h) gcn[nf][h] = bcol(wn + 8 * nf + 2 * q + h);
#pragma unroll
  for (int mf = 0; mf < 4; ++mf) {
    const int m = wm + 8 * mf + g, gr = brow(ti, m);
    if (gr < 0) continue;
    if (ZP) {
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (gcn[nf][h] >= 0) Zm[(int64_t)gcn[nf][h] * ld + gr] = acc[mf][nf][h];
    } else if (kUpdRed) {
      // C += (-acc) as L2 reductions (no return value, no load latency in the task): the block
      // has exactly one writer at a time (tile counters), so the result is the same rounded
      // difference C - acc and the order of updates per entry stays the task order
      const int tr = ti + (m >> 5);
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = wn + 8 * nf + 2 * q + h, tc = tj + (n >> 5);
          if (gcn[nf][h] >= 0 && !(tr < tc || (tr == tc && (m & 31) < (n & 31))))
            asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(Fm + (int64_t)gcn[nf][h] * ld + gr),
                         "d"(-acc[mf][nf][h]) : "memory");
        }
    } else {
      double cv[NF][2];
      bool ok[NF][2];
      const int tr = ti + (m >> 5);
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = wn + 8 * nf + 2 * q + h, tc = tj + (n >> 5);
          ok[nf][h] = gcn[nf][h] >= 0 && !(tr < tc || (tr == tc && (m & 31) < (n & 31)));
          cv[nf][h] = ok[nf][h] ? __ldcg(Fm + (int64_t)gcn[nf][h] * ld + gr) : 0.0;
        }
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (ok[nf][h]) Fm[(int64_t)gcn[nf][h] * ld + gr] = cv[nf][h] - acc[mf][nf][h];
    }
  }
}

// One block Z(t, cb) of the solve panel Z = [I; L21] L11^{-1} (L11 unit lower, the 2x2
// pivot slots belong to D), t a tile of the split grid, cb a pivot column block:
//   pivot tile t < P:   Z(t, cb) = L(t,t)^{-1} (delta_{t,cb} I - sum_{j=cb}^{t-1} L(t,j) Z(j,cb))
//   struct tile t >= P: Z(t, cb) = sum_{j=cb}^{P-1} L(t,j) Z(j,cb)
// Pivot rows go top-down, so block (t, cb) needs only D_t and the tiles above it in its
// column block: the panel of a front's pivot tile t is built while steps > t are still
// being factored, and the last one is one task after the front's last pivot step.  The
// sum is on DMMA; the left solve with L(t,t) is trsm_rows on the transposed block
// against the published L^T of step t.  Block (t, t) also publishes the factored diagonal
// block from scratch into F.  Returns the transposed block in S.b[0] (Pw[col][row]).
__device__ void f_ztask_pre(const sgn::FactorArgs& A, const DFront& F, int b, int t, int cb, Smem& S) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int npiv = F.npiv, P = sgn::ptiles(npiv);
  const int lo = sgn::tile_lo(npiv, t), nr = sgn::tile_hi(npiv, F.nrow, t) - lo;
  const bool piv = t < P;
  const int64_t ld = sgn::front_ld(F.nrow);
  double* Fm = front_ptr(A, F, b);
  const double* Zm = A.zstore + (int64_t)b * A.zstride + F.zoff;
  const double* ds = A.dscr + (int64_t)b * A.dstride + F.doff;
  int* cf = A.cnt + (int64_t)b * A.n_fcnt + F.cbase;
  const int Tn = sgn::ntiles_front(npiv, F.nrow);
  const int c0 = cb * kTile, wb = min(kTile, npiv - c0);
  double (*Pw)[kTile + 1] = v33(S.b[0]);
  V40 Lk = v40(S.b[2]);     // K-major: Lk[kk][row] = L(lo + row, k0 + kk)
  V40 Zk = v40(S.b[3]);     // K-major: Zk[kk][col] = Z(k0 + kk, c0 + col)
  const int row0 = warp * 8, i = row0 + g;
  double acc[4][2];
#pragma unroll
  for (int nf = 0; nf < 4; ++nf) acc[nf][0] = acc[nf][1] = 0.0;
  // L(t, j) is final up front (pivot tiles: DIAG(t) implies every panel of steps < t that
  // wrote row tile t; struct tiles: the last step's panels, PAN(P-1), imply all earlier
  // ones).  The Z(j, cb) terms are consumed as they become final (progressive waits on
  // ZC(cb) instead of one up-front wait for the whole column above t): the column chain
  // Z(t-1, cb) -> Z(t, cb) then costs one term, not the whole sum.
  __shared__ int s_ready;
  const int jend = piv ? t : P;
  int ready = cb;
  if (tid == 0) {
    if (piv) spin_ge(cf + sgn::cnt_diag(P, t), 1);
    else spin_ge(cf + sgn::cnt_pan(P - 1), sgn::panel_tasks(npiv, F.nrow, P - 1));
  }
  __syncthreads();
  double vl[8], vz[8];
#define SGN_Z_LOAD(J_)                                                                              \
  do {                                                                                              \
    const int k0_ = (J_) * kTile, kw_ = min(kTile, npiv - k0_);                                     \
    _Pragma("unroll") for (int u = 0; u < 8; ++u) {                                                 \
      const int e = tid + u * kFThreads;                                                            \
      const int r = e & 31, c = e >> 5;                                                             \
      vl[u] = (r < nr && c < kw_) ? __ldcg(Fm + (int64_t)(k0_ + c) * ld + lo + r) : 0.0;            \
      vz[u] = (r < kw_ && c < wb) ? __ldcg(Zm + (int64_t)(c0 + c) * ld + k0_ + r) : 0.0;            \
    }                                                                                               \
  } while (0)
  auto wait_term = [&](int j) {
    if (j < ready) return;
    if (tid == 0) {
      int zc;
      while ((zc = ld_acq(cf + sgn::cnt_zc(P, Tn, cb))) < j - cb + 1) __nanosleep(20);
      s_ready = cb + zc;
    }
    __syncthreads();
    ready = s_ready;
  };
  if (cb < jend) {
    wait_term(cb);
    SGN_Z_LOAD(cb);
  }
  for (int j = cb; j < jend; ++j) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * kFThreads;
      const int r = e & 31, c = e >> 5;
      Lk[c][r] = vl[u];
      Zk[r][c] = vz[u];
    }
    __syncthreads();
    if (j + 1 < jend) {                   // next term's tiles in flight during the DMMAs
      wait_term(j + 1);
      SGN_Z_LOAD(j + 1);
    }
#pragma unroll
    for (int kk = 0; kk < kTile; kk += 4) {
      const double a = Lk[kk + q][row0 + g];
#pragma unroll
      for (int nf = 0; nf < 4; ++nf) dmma_8x8x4(acc[nf][0], acc[nf][1], a, Zk[kk + q][nf * 8 + g]);
    }
    __syncthreads();
  }
#undef SGN_Z_LOAD
  if (piv) {                // the left solve: D_t / L^T of step t (DIAG(t) waited above)
    if (cb == t) {          // block (t, t) also publishes the factored diagonal block into F
      const double* blk = ds + (int64_t)t * sgn::kDiagStride;
      for (int e = tid; e < kTile * kTile; e += kFThreads) {
        const int ii = e >> 5, jj = e & 31;
        if (ii < nr && jj < nr && ii >= jj) Fm[(int64_t)(lo + jj) * ld + lo + ii] = __ldcg(blk + e);
      }
    }
    double (*Lt)[kTile + 1] = v33(S.b[1]);
    const double* lt = ds + (int64_t)t * sgn::kDiagStride + kTile * kTile;
    for (int e = tid; e < kTile * kTile; e += kFThreads) Lt[e >> 5][e & 31] = __ldcg(lt + e);
  }
#pragma unroll
  for (int nf = 0; nf < 4; ++nf)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = nf * 8 + 2 * q + h;
      double v = 0.0;
      if (i < nr && j < wb) v = piv ? (((cb == t && i == j) ? 1.0 : 0.0) - acc[nf][h]) : acc[nf][h];
      Pw[j][i] = v;
    }
}

__device__ void f_ztask_post(const sgn::FactorArgs& A, const DFront& F, int b, int t, int cb, Smem& S) {
  const int tid = threadIdx.x;
  const int lo = sgn::tile_lo(F.npiv, t), nr = sgn::tile_hi(F.npiv, F.nrow, t) - lo;
  const int64_t ld = sgn::front_ld(F.nrow);
  double* Zm = A.zstore + (int64_t)b * A.zstride + F.zoff;
  const int c0 = cb * kTile, wb = min(kTile, F.npiv - c0);
  double (*Pw)[kTile + 1] = v33(S.b[0]);
  for (int e = tid; e < kTile * kTile; e += kFThreads) {
    const int ii = e & 31, c = e >> 5;
    if (ii < nr && c < wb) Zm[(int64_t)(c0 + c) * ld + lo + ii] = Pw[c][ii];
  }
}

__global__ void __launch_bounds__(kFThreads, 4)
k_factor_dag(const sgn::FactorArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  __shared__ int s_idx, s_base, s_left, s_sub, s_subend, s_cur;
  const int64_t total = A.ntask * A.batch;
  const int tid = threadIdx.x;
  // batched factorizations take runs of A.run consecutive instances of one task per grab
  // (one atomic and one look at the task list per run); the run is processed in order, so
  // the earliest unfinished task is still always running (deadlock freedom unchanged).
  // An F_FAT task (a whole small front) runs its sub-tasks fat[a .. b) back to back under
  // the same index before the next grab.
  if (tid == 0) { s_left = 0; s_sub = 0; s_subend = 0; s_idx = -1; }
  const bool retiring = (int)blockIdx.x >= A.retire_from;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      if (s_sub < s_subend) {
        s_cur = s_sub++;
      } else if (retiring && s_left == 0 && s_idx >= A.retire_at) {
        s_idx = INT_MAX;                     // leave: the slot goes to the concurrent launch
        s_cur = -1;
      } else {
        if (s_left == 0) { s_base = atomicAdd(A.head, A.run); s_left = A.run; }
        s_idx = s_base + (A.run - s_left);
        --s_left;
        s_cur = -1;
      }
    }
    __syncthreads();
    const int64_t idx = s_idx;
    if (idx >= total) return;
    const int64_t tix = idx / A.batch;
    const int b = (int)(idx - tix * A.batch);
    sgn::FTask T = (s_cur >= 0) ? A.fat[s_cur] : A.tasks[tix];
    if ((T.kind_k & 7) == sgn::F_FAT) {
      __syncthreads();                                        // s_cur read by every thread
      if (tid == 0) { s_sub = T.a + 1; s_subend = T.b; }
      T = A.fat[T.a];
    }
    const int kind = T.kind_k & 7, k = T.kind_k >> 3;
    const DFront F = A.fronts[T.f];
    int* cnt = A.cnt + (int64_t)b * A.n_fcnt;
    int* cf = cnt + F.cbase;
    const int P = sgn::ptiles(F.npiv);
    if (tid == 0) {
      S.tr = A.trace ? A.trace + idx * 8 : nullptr;
      if (S.tr) S.tr[0] = gtimer();
    }
    const int Tn = sgn::ntiles_front(F.npiv, F.nrow);
    // F_UPDATE: b = tj | (ns << 16) applies steps k-ns+1 .. k (ns = 0 or 1: step k alone)
    // F_UPD2: bit 15 of b = one column tile (rows paired only)
    const bool u2single = (kind == sgn::F_UPD2) && (T.b & 0x8000);
    const int tjb = (kind == sgn::F_UPD2) ? (T.b & 0x7fff) : (T.b & 0xffff);
    const int ns = (kind == sgn::F_UPDATE || kind == sgn::F_UPD2) ? max(1, T.b >> 16) : 1;
    const int tjw = u2single ? 1 : 2;       // column tiles of an F_UPD2 block
    // the task's dependency counters, one per lane of warp 0: the acquire loads of up to 8
    // counters are in flight together instead of one L2 round trip after another (the
    // barrier below orders every thread of the CTA after all of them)
    if (tid < 32) {
      const int lane = tid;
      if (kind == sgn::F_ASM) {
        for (int ci = F.child_begin + lane; ci < F.child_end; ci += 32) {
          const DFront C = A.fronts[A.children[ci]];
          spin_ge(cnt + C.cbase, C.ftotal);
        }
      } else if (kind == sgn::F_PANEL) {          // DIAG(k) is awaited inside (after P loads)
        if (T.a == 0) {
          if (lane == 0) spin_ge(cf + sgn::cnt_tile(P, k + 1, k), 1 + k);
        } else if (lane < 4) {
          const int i = k + 2 + 4 * (T.a - 1) + lane;
          if (i < Tn) spin_ge(cf + sgn::cnt_tile(P, i, k), 1 + k);
        }
      } else if (kind == sgn::F_UPDATE || kind == sgn::F_DIAGUPD) {   // PAN(k) awaited inside
        const int ti = (kind == sgn::F_DIAGUPD) ? k + 1 : T.a, tj = (kind == sgn::F_DIAGUPD) ? k + 1 : tjb;
        if (lane == 0) spin_ge(cf + sgn::cnt_tile(P, ti, tj), 2 + k - ns);
      } else if (kind == sgn::F_ZPAN2) {          // L final (last step's TRSMs), both Z columns complete
        if (lane == 0) spin_ge(cf + sgn::cnt_pan(P - 1), sgn::panel_tasks(F.npiv, F.nrow, P - 1));
        if (lane == 1) spin_ge(cf + sgn::cnt_zc(P, Tn, T.b), P - T.b);
        if (lane == 2 && T.b + 1 < P) spin_ge(cf + sgn::cnt_zc(P, Tn, T.b + 1), P - T.b - 1);
      } else if (kind == sgn::F_UPD2) {           // every tile of the block, then the TRSMs of step k
        if (lane < 4) {
          const int x = T.a + (lane >> 1), y = tjb + (lane & 1);
          if (x < min(T.a + 2, Tn) && y < min(tjb + tjw, Tn) && x >= y) spin_ge(cf + sgn::cnt_tile(P, x, y), 2 + k - ns);
        } else if (lane < 6 + tjw) {
          const int x = lane - 4;
          const int t = (x < 2) ? T.a + x : tjb + x - 2;
          if (t < Tn) spin_ge(cf + sgn::cnt_pant(F.npiv, F.nrow, k, sgn::pan_task_of(k, t)), 1);
        }
      }                                           // Z(t, cb): progressive waits in f_ztask_pre
    }
    __syncthreads();
    if (A.trace && tid == 0) A.trace[idx * 8 + 1] = gtimer();
    // phase 1: kind-specific work; the heavy unrolled kernels (pivot-block LDL^T and the
    // row substitution) then run from ONE call site each (instruction-cache footprint)
    int fac_k = -1, nr_trsm = 0;
    double (*fac_tile)[kTile + 1] = v33(S.a);
    double (*tr_p)[kTile + 1] = v33(S.b[0]);
    double (*tr_l)[kTile + 1] = v33(S.a);
    if (kind == sgn::F_ASM) {
      if (k == 1) f_asm2(A, F, b, T.a, T.b, S);
      else f_asm(A, F, b, T.a, T.b, S);
      if (T.a == 0 && T.b == 0 && F.npiv > 0) fac_k = 0;
    } else if (kind == sgn::F_PANEL) {
      nr_trsm = f_panel_pre(A, F, b, k, T.a, S);
      tr_p = v33(S.b[tid >> 5]);
    } else if (kind == sgn::F_UPDATE || kind == sgn::F_DIAGUPD) {
      const bool dg = (kind == sgn::F_DIAGUPD);
      f_update(A, F, b, k - ns + 1, k, dg ? k + 1 : T.a, dg ? k + 1 : tjb, S, dg);
      if (dg) { fac_k = k + 1; fac_tile = v33(S.b[1]); }
    } else if (kind == sgn::F_UPD2) {
      if (u2single) f_block64<false, 32>(A, F, b, k - ns + 1, k, T.a, tjb, S);
      else f_block64<false, 64>(A, F, b, k - ns + 1, k, T.a, tjb, S);
    } else if (kind == sgn::F_ZPAN2) {
      f_block64<true, 64>(A, F, b, T.b, P - 1, T.a, T.b, S);
    } else {
      f_ztask_pre(A, F, b, T.a, T.b, S);
      nr_trsm = (T.a < P && tid < 32) ? 32 : 0;
      tr_l = v33(S.b[1]);
    }
    if (fac_k >= 0) factor_publish(A, F, b, fac_k, fac_tile, S);
    __syncthreads();
    if (kind == sgn::F_PANEL) tmark(S, 4);
    if (nr_trsm > 0) trsm_rows(tr_p, tr_l);
    __syncthreads();
    tmark(S, 7);
    if (kind == sgn::F_PANEL) f_panel_post(A, F, b, k, T.a, nr_trsm, S);
    else if (kind == sgn::F_ZPANEL) f_ztask_post(A, F, b, T.a, T.b, S);
    __syncthreads();   // every thread's writes precede the release
    if (tid == 0) {
      int* s1;
      int* s2 = cf;                                            // DONE
      int* s3 = nullptr;
      if (kind == sgn::F_ZPANEL) { s1 = (T.a < P) ? cf + sgn::cnt_zc(P, Tn, T.b) : nullptr; s2 = nullptr; }
      else if (kind == sgn::F_ZPAN2) { s1 = nullptr; s2 = nullptr; }
      else if (kind == sgn::F_PANEL) {
        s1 = cf + sgn::cnt_pan(k);
        s3 = cf + sgn::cnt_pant(F.npiv, F.nrow, k, T.a);
      }
      else if (kind == sgn::F_DIAGUPD) { s1 = cf + sgn::cnt_tile(P, k + 1, k + 1); s3 = cf + sgn::cnt_diag(P, k + 1); }
      else if (kind == sgn::F_UPD2) {
        s1 = nullptr;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int x = T.a; x < min(T.a + 2, Tn); ++x)
          for (int y = tjb; y < min(tjb + tjw, Tn); ++y)
            if (x >= y) asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(cf + sgn::cnt_tile(P, x, y)), "r"(ns) : "memory");
      }
      else if (kind == sgn::F_ASM && k == 1) {   // every lower tile of the 64x64 block
        s1 = nullptr;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int x = T.a; x < min(T.a + 2, Tn); ++x)
          for (int y = tjb; y < min(tjb + 2, Tn); ++y)
            if (x >= y) asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(cf + sgn::cnt_tile(P, x, y)) : "memory");
        if (T.a == 0 && T.b == 0 && F.npiv > 0) s3 = cf + sgn::cnt_diag(P, 0);
      }
      else {
        s1 = cf + sgn::cnt_tile(P, T.a, tjb);
        if (kind == sgn::F_ASM && T.a == 0 && T.b == 0 && F.npiv > 0) s3 = cf + sgn::cnt_diag(P, 0);
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      if (s1) asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(s1), "r"(ns) : "memory");   // TILE += steps applied
      if (s2) asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(s2) : "memory");
      if (s3) asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(s3) : "memory");
    }
    if (A.trace && tid == 0) {
      A.trace[idx * 8 + 2] = gtimer();
      A.trace[idx * 8 + 3] = smid();
    }
  }
}

}  // namespace

namespace sgn {

int factor_dag_grid() {
  static int cached_dev = -1, sms = 0, occ = 0;     // one device per process
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev != cached_dev) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    if (cudaFuncSetAttribute(k_factor_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_factor_dag, kFThreads, sizeof(Smem)) != cudaSuccess) return 0;
    cached_dev = dev;
  }
  int per_sm = std::max(occ, 1);
  return sms * per_sm;
}

int launch_factor_dag(const FactorArgs& A, int grid, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = A.ntask * A.batch;
  if (total == 0) return SGN_OK;
  cudaError_t e = cudaMemsetAsync(A.head, 0, (size_t)(1 + A.batch * A.n_fcnt) * sizeof(int), st);
  if (e != cudaSuccess) { last_error() = std::string("counter reset: ") + cudaGetErrorString(e); return SGN_CUDA_ERROR; }
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid, (total + A.run - 1) / A.run));
  count_launch();
  k_factor_dag<<<g, kFThreads, sizeof(Smem), st>>>(A);
  e = cudaGetLastError();
  if (e != cudaSuccess) { last_error() = std::string("k_factor_dag: ") + cudaGetErrorString(e); return SGN_CUDA_ERROR; }
  return SGN_OK;
}

}  // namespace sgn
