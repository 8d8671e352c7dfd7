// Device numeric phase of the SGN KKT solver on B200 (sm_100a) + the C ABI.
//
// Replaces, on the GPU, the reference's SuperLU numeric LU (spla.splu, reference
// pkg/src/sgnopt/linear_solvers.py:87), its triangular solves (linear_solvers.py:93-97),
// the stabilization (linear_solvers.py:111-127), the relative-residual SpMV
// (linear_solvers.py:105-108) and the BiCGSTAB refinement (linear_solvers.py:130-211).
//
// Factorization: multifrontal LDL^T over the host-built assembly tree (symbolic.cpp).
// Per tree level: (1) tile-owner assembly of all fronts of the level (original entries +
// stabilization shift + fixed-order extend-add of children update matrices -- atomic
// free, bitwise deterministic); (2) per 32-column panel: a panel kernel (redundant
// in-smem LDL^T of the diagonal block with 2x2 / 1x1 pivots + TRSM of a 32-row tile)
// and a Schur-update kernel whose 32x32 tiles run on the FP64 tensor pipe
// (mma.sync.m8n8k4.f64 -> DMMA).  Solves are level-scheduled, one CTA per front,
// warp-shuffle diagonal blocks.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sgn_b200.h"
#include "sgn_internal.h"

using sgn::DFront;
using sgn::kTile;
using sgn::kPanelTiles;
using sgn::Work;

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      sgn::last_error() = std::string(#expr) + ": " + cudaGetErrorString(_e);       \
      return SGN_CUDA_ERROR;                                                        \
    }                                                                               \
  } while (0)

namespace {

constexpr int kAsmThreads = 256;
constexpr int kPanelThreads = 128;
constexpr int kUpdThreads = 128;
constexpr int kSolveThreads = 256;

// ------------------------------------------------------------------------------------
// assembly: one CTA owns one 32x32 lower tile of one front
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kAsmThreads)
k_assemble(const Work* __restrict__ work, const DFront* __restrict__ fronts,
           const int32_t* __restrict__ children, const int32_t* __restrict__ rel,
           const int64_t* __restrict__ tile_ptr, const int64_t* __restrict__ tile_nnz,
           const int32_t* __restrict__ tile_loc, const int8_t* __restrict__ kind_pos,
           const double* __restrict__ values, int64_t vstride, double eps_x, double eps_l,
           const double* __restrict__ eps_xv, const double* __restrict__ eps_lv,
           double* __restrict__ fstore, int64_t fstride) {
  __shared__ double tile[kTile][kTile + 1];
  const Work w = work[blockIdx.x];
  const int b = blockIdx.y;
  const DFront F = fronts[w.f];
  const int ti = w.a, tj = w.b;
  const int tid = threadIdx.x;
  double* fb = fstore + (int64_t)b * fstride;
  const double* vals = values + (int64_t)b * vstride;
  for (int e = tid; e < kTile * kTile; e += blockDim.x) tile[e >> 5][e & 31] = 0.0;
  __syncthreads();
  const int64_t tid_g = F.tile_base + (int64_t)ti * (ti + 1) / 2 + tj;
  {
    const int64_t e0 = tile_ptr[tid_g], e1 = tile_ptr[tid_g + 1];
#pragma unroll 4
    for (int64_t e = e0 + tid; e < e1; e += kAsmThreads) {
      const int loc = tile_loc[e];
      tile[loc >> 5][loc & 31] = vals[tile_nnz[e]];
    }
  }
  __syncthreads();
  if (ti == tj && tid < kTile) {
    const int r = ti * kTile + tid;
    if (r < F.npiv) {
      const int8_t k = kind_pos[F.first + r];
      if (k == 1) tile[tid][tid] += eps_xv ? eps_xv[b] : eps_x;
      else if (k == 2) tile[tid][tid] -= eps_lv ? eps_lv[b] : eps_l;
    }
  }
  const int i0 = ti * kTile, i1 = min(i0 + kTile, F.nrow);
  const int j0 = tj * kTile, j1 = min(j0 + kTile, F.nrow);
  for (int ci = F.child_begin; ci < F.child_end; ++ci) {
    const DFront C = fronts[children[ci]];
    const int cn = C.nrow - C.npiv;
    if (cn == 0) continue;
    const int32_t* rc = rel + C.rel_off;
    const int r_lo = lower_bound_i32(rc, cn, i0), r_hi = lower_bound_i32(rc, cn, i1);
    const int s_lo = lower_bound_i32(rc, cn, j0), s_hi = lower_bound_i32(rc, cn, j1);
    const int nr = r_hi - r_lo, ns = s_hi - s_lo;
    __syncthreads();
    if (nr > 0 && ns > 0) {
      const double* U = fb + C.foff;
      const int64_t ldc = C.nrow;
#pragma unroll 4
      for (int idx = tid; idx < nr * ns; idx += kAsmThreads) {
        const int r = r_lo + idx % nr, s = s_lo + idx / nr;
        if (r >= s) {
          const double u = U[(int64_t)(C.npiv + s) * ldc + C.npiv + r];
          tile[rc[r] - i0][rc[s] - j0] += u;
        }
      }
    }
  }
  __syncthreads();
  double* Fm = fb + F.foff;
  const int64_t ld = F.nrow;
  for (int e = tid; e < kTile * kTile; e += blockDim.x) {
    const int ii = e & 31, jj = e >> 5;
    const int gi = i0 + ii, gj = j0 + jj;
    if (gi < i1 && gj < j1) Fm[(int64_t)gj * ld + gi] = tile[ii][jj];
  }
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// ------------------------------------------------------------------------------------
// One warp factors a <= 32 x 32 diagonal block held in shared memory (lane i owns row i):
// LDL^T with 2x2 pivots on (2t, 2t+1) (pivtype 2) or 1x1 pivots; D stays in place, L below
// the pivot blocks.  Rows live in registers; columns are exchanged with shuffles.
// ------------------------------------------------------------------------------------
// One warp factors the <= 32 x 32 diagonal block with rows in registers (lane i = row i).
// Every shuffle is executed by all lanes (no divergent branch around it, so the compiler
// emits native SHFL); inactive steps/rows are masked with selects.  Templated on the
// pivot type so each instantiation stays small (~2k instructions).
template <int PT>
__device__ __forceinline__ void warp_ldlt_reg(double (*D)[kTile + 1], int w, int* bad, bool store) {
  const int i = threadIdx.x & 31;
  int first_bad = 1 << 30;
  double d[kTile];
#pragma unroll
  for (int k = 0; k < kTile; ++k) d[k] = (k <= i) ? D[i][k] : 0.0;
#pragma unroll
  for (int j = 0; j < kTile; j += PT) {
    const bool act = (j < w);
    if (PT == 2) {
      const double a = __shfl_sync(0xffffffffu, d[j], j);
      const double bb = __shfl_sync(0xffffffffu, d[j], j + 1);
      const double c = __shfl_sync(0xffffffffu, d[j + 1], j + 1);
      double det = a * c - bb * bb;
      first_bad = (act && (det == 0.0 || !isfinite(det)) && first_bad > j) ? j : first_bad;
      det = act ? det : 1.0;
      const double rdet = 1.0 / det;
      const double ia = c * rdet, ib = -bb * rdet, ic = a * rdet;
      const bool below = act && (i > j + 1) && (i < w);
      const double x0 = d[j], x1 = d[j + 1];
      const double l0 = below ? x0 * ia + x1 * ib : 0.0;
      const double l1 = below ? x0 * ib + x1 * ic : 0.0;
#pragma unroll
      for (int k = j + 2; k < kTile; ++k) {
        const double y0 = __shfl_sync(0xffffffffu, x0, k);
        const double y1 = __shfl_sync(0xffffffffu, x1, k);
        const double nd = d[k] - (l0 * y0 + l1 * y1);
        d[k] = (below && k <= i) ? nd : d[k];
      }
      d[j] = below ? l0 : d[j];
      d[j + 1] = below ? l1 : d[j + 1];
    } else {
      double dj = __shfl_sync(0xffffffffu, d[j], j);
      first_bad = (act && (dj == 0.0 || !isfinite(dj)) && first_bad > j) ? j : first_bad;
      dj = act ? dj : 1.0;
      const bool below = act && (i > j) && (i < w);
      const double x = d[j];
      const double l = below ? x / dj : 0.0;
#pragma unroll
      for (int k = j + 1; k < kTile; ++k) {
        const double y = __shfl_sync(0xffffffffu, x, k);
        const double nd = d[k] - l * y;
        d[k] = (below && k <= i) ? nd : d[k];
      }
      d[j] = below ? l : d[j];
    }
  }
  __syncthreads();   // all warps have read D before warp 0 overwrites it
  if (store) {
#pragma unroll
    for (int k = 0; k < kTile; ++k) if (k <= i) D[i][k] = d[k];
    if (i == 0 && first_bad < (1 << 30)) atomicMin(bad, first_bad);
  }
}

// TRSM of one 32-row tile (lane = row, row in registers): W L11^T = P, right-looking so
// the FMAs of a step are independent; L11 columns are broadcast reads from smem.
template <int PT>
__device__ __forceinline__ void warp_trsm_reg(double (*P)[kTile + 1], const double (*D)[kTile + 1]) {
  const int i = threadIdx.x & 31;
  double p[kTile];
#pragma unroll
  for (int c = 0; c < kTile; ++c) p[c] = P[i][c];
#pragma unroll
  for (int cp = 0; cp < kTile; ++cp) {
#pragma unroll
    for (int c = cp + 1; c < kTile; ++c) {
      if (PT == 2 && (cp & 1) == 0 && c == cp + 1) continue;   // D slot, compile-time
      p[c] -= p[cp] * D[c][cp];
    }
  }
#pragma unroll
  for (int c = 0; c < kTile; ++c) P[i][c] = p[c];
}

// Panel step k of a front: every CTA factors the diagonal block (one warp, registers +
// smem; a few us), CTA t == 0 stores L11/D and the block inverse, CTAs t >= 1 form their
// 32-row tile of W = P L11^{-T} on DMMA and L21 = W D^{-1}.
template <int PT>
__global__ void __launch_bounds__(kPanelThreads, 1)
k_panel(const Work* __restrict__ work, const DFront* __restrict__ fronts,
        const int64_t* __restrict__ perm, double* __restrict__ fstore, int64_t fstride,
        double* __restrict__ wstore, int64_t wstride, double* __restrict__ dscr, int64_t dstride,
        long long* __restrict__ status) {
  __shared__ double D[kTile][kTile + 1];
  __shared__ double P[kPanelTiles][kTile][kTile + 1];
  __shared__ double Dinv[kTile][3];      // per pivot block: (ia, ib, ic) or (1/d)
  __shared__ int bad;
  const Work wk = work[blockIdx.x];
  const int b = blockIdx.y;
  const DFront F = fronts[wk.f];
  const int j0 = wk.a * kTile;
  const int w = min(kTile, F.npiv - j0);
  const int t = wk.b;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  double* Fm = fstore + (int64_t)b * fstride + F.foff;
  const int64_t ld = F.nrow;
  if (tid == 0) bad = 1 << 30;
#pragma unroll
  for (int e = tid; e < kTile * kTile; e += kPanelThreads) {   // loads all in flight
    const int i = e & 31, j = e >> 5;
    D[i][j] = (i < w && j < w && i >= j) ? Fm[(int64_t)(j0 + j) * ld + j0 + i] : 0.0;
  }
  // this CTA: row tiles t .. t+3 below the diagonal block, warp w owns tile t+w
  const int r0 = j0 + w + (t - 1 + warp) * kTile;
  const int nr = (t > 0) ? max(0, min(kTile, F.nrow - r0)) : 0;
  double (*Pw)[kTile + 1] = P[warp];
  if (t > 0) {
    double v[kTile];
#pragma unroll
    for (int j = 0; j < kTile; ++j) v[j] = (lane < nr && j < w) ? Fm[(int64_t)(j0 + j) * ld + r0 + lane] : 0.0;
#pragma unroll
    for (int j = 0; j < kTile; ++j) Pw[lane][j] = v[j];
  }
  __syncthreads();
  warp_ldlt_reg<PT>(D, w, &bad, warp == 0);   // every warp runs it (converged shuffles);
  __syncthreads();                             // only warp 0 stores the result
  if (tid < w) {
    if (PT == 2) {
      if ((tid & 1) == 0) {
        const double a = D[tid][tid], bb = D[tid + 1][tid], cc = D[tid + 1][tid + 1];
        const double rdet = 1.0 / (a * cc - bb * bb);
        Dinv[tid][0] = cc * rdet; Dinv[tid][1] = -bb * rdet; Dinv[tid][2] = a * rdet;
      }
    } else {
      Dinv[tid][0] = 1.0 / D[tid][tid];
    }
  }
  __syncthreads();
  if (t == 0) {
    // the factored block goes to scratch: other CTAs of this launch may still be reading
    // the unfactored block from F (k_zpanel copies it into F at the end of the level)
    if (tid == 0 && bad < (1 << 30)) atomicMin(&status[b], (long long)perm[F.first + j0 + bad]);
    double* ds = dscr + (int64_t)b * dstride + F.doff + (int64_t)wk.a * kTile * kTile;
    for (int e = tid; e < kTile * kTile; e += blockDim.x) ds[e] = D[e >> 5][e & 31];
    return;
  }
  // W = P L11^{-T} by row-wise substitution (lane per row of the warp's tile, row in
  // registers, right-looking so the FMAs are independent; explicit inverses would
  // amplify rounding in the factor itself)
  if (nr > 0) warp_trsm_reg<PT>(Pw, D);   // W = P L11^{-T}: substitution, no explicit inverse
  __syncwarp();
  if (nr == 0) return;
  double* Wb = wstore + (int64_t)b * wstride + F.woff + (int64_t)(t - 1 + warp) * kTile * kTile;
  for (int e = lane; e < nr * kTile; e += 32) {
    const int i = e / kTile, c = e % kTile;
    Wb[(int64_t)i * kTile + c] = (c < w) ? Pw[i][c] : 0.0;
  }
  // L21 = W D^{-1} with the pivot-block inverses precomputed in Dinv (no divisions here)
  for (int e = lane; e < kTile * kTile; e += 32) {
    const int i = e & 31, c = e >> 5;
    if (i >= nr || c >= w) continue;
    double l;
    if (PT == 2) {
      const int c0 = c & ~1;
      const double x0 = Pw[i][c0], x1 = Pw[i][c0 + 1];
      l = (c == c0) ? x0 * Dinv[c0][0] + x1 * Dinv[c0][1] : x0 * Dinv[c0][1] + x1 * Dinv[c0][2];
    } else {
      l = Pw[i][c] * Dinv[c][0];
    }
    Fm[(int64_t)(j0 + c) * ld + r0 + i] = l;
  }
}

// ------------------------------------------------------------------------------------
// Schur update of one 32x32 lower tile of the trailing matrix on the FP64 tensor pipe:
//   C[i, j] -= sum_c L21[i, c] * W[j, c]       (W = L21 D, row-major scratch)
// mma.sync.aligned.m8n8k4.row.col.f64: A 8x4 (row), B 4x8 (col), C 8x8.
// ------------------------------------------------------------------------------------

__global__ void __launch_bounds__(kUpdThreads)
k_update(const Work* __restrict__ work, const DFront* __restrict__ fronts,
         double* __restrict__ fstore, int64_t fstride, const double* __restrict__ wstore,
         int64_t wstride) {
  __shared__ double As[kTile][kTile + 1];
  __shared__ double Bs[kTile][kTile + 1];
  const Work wk = work[blockIdx.x];
  const int b = blockIdx.y;
  const DFront F = fronts[wk.f];
  const int j0 = wk.a * kTile;
  const int w = min(kTile, F.npiv - j0);
  const int o = j0 + w;
  const int ti = wk.b, tj = wk.c;
  const int rbase = o + ti * kTile, cbase = o + tj * kTile;
  const int nr = min(kTile, F.nrow - rbase), nc = min(kTile, F.nrow - cbase);
  const int tid = threadIdx.x;
  double* Fm = fstore + (int64_t)b * fstride + F.foff;
  const int64_t ld = F.nrow;
  const double* Wb = wstore + (int64_t)b * wstride + F.woff;
#pragma unroll
  for (int e = tid; e < kTile * kTile; e += kUpdThreads) {
    const int i = e & 31, c = e >> 5;
    As[i][c] = (i < nr && c < w) ? Fm[(int64_t)(j0 + c) * ld + rbase + i] : 0.0;
  }
#pragma unroll
  for (int e = tid; e < kTile * kTile; e += kUpdThreads) {
    const int c = e & 31, j = e >> 5;
    Bs[j][c] = (j < nc && c < w) ? Wb[(int64_t)(tj * kTile + j) * kTile + c] : 0.0;
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int row0 = warp * 8;
  double acc[4][2];
#pragma unroll
  for (int nf = 0; nf < 4; ++nf) acc[nf][0] = acc[nf][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < kTile; kk += 4) {
    const double a = As[row0 + g][kk + q];
#pragma unroll
    for (int nf = 0; nf < 4; ++nf) {
      const double bv = Bs[nf * 8 + g][kk + q];
      dmma_8x8x4(acc[nf][0], acc[nf][1], a, bv);
    }
  }
  const int i = row0 + g;
  if (i < nr) {
#pragma unroll
    for (int nf = 0; nf < 4; ++nf) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = nf * 8 + 2 * q + h;
        if (j < nc && (ti != tj || i >= j)) Fm[(int64_t)(cbase + j) * ld + rbase + i] -= acc[nf][h];
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// level-scheduled multifrontal solves (one CTA per front)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ bool pair_skip(int pivtype, int row, int col) {
  // in 2x2-pivot fronts L(2t+1, 2t) is structurally zero (slot holds D)
  return pivtype == 2 && (col & 1) == 0 && row == col + 1;
}

// ------------------------------------------------------------------------------------
// Solve panel Z = [I; L21] L11^{-1} of one front (rows r0..r0+31), built after the front
// is factored: Z L11 = B with B = e_r (pivot rows) or L21 (struct rows), swept right to
// left in 32-column blocks; the inter-block products run on DMMA.  With Z the
// triangular solves are one parallel pass per front (k_fwd / k_bwd below).
// ------------------------------------------------------------------------------------
constexpr int kZThreads = 256;
__global__ void __launch_bounds__(kZThreads)
k_zpanel(const Work* __restrict__ work, const DFront* __restrict__ fronts,
         double* __restrict__ fstore, int64_t fstride, double* __restrict__ zstore,
         int64_t zstride, const double* __restrict__ dscr, int64_t dstride) {
  __shared__ double Ts[kTile][kTile + 1];          // final Z block of the step (rows x cols)
  __shared__ double Ls[kTile][kTile + 1];          // diagonal block of L11
  const Work wk = work[blockIdx.x];
  const int b = blockIdx.y;
  const DFront F = fronts[wk.f];
  const int r0 = wk.a;
  const int nr = min(kTile, F.nrow - r0);
  const int npiv = F.npiv;
  const int64_t ld = F.nrow;
  double* Fm = fstore + (int64_t)b * fstride + F.foff;
  double* Zm = zstore + (int64_t)b * zstride + F.zoff;
  const double* ds = dscr + (int64_t)b * dstride + F.doff;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int cmax = (r0 < npiv) ? min(npiv, r0 + nr) : npiv;
  if (r0 < npiv) {   // this row tile owns diagonal block r0/32: publish the factored block to F
    const double* blk = ds + (int64_t)(r0 / kTile) * kTile * kTile;
    const int wd = min(kTile, npiv - r0);
    for (int e = tid; e < kTile * kTile; e += blockDim.x) {
      const int i = e >> 5, j = e & 31;
      if (i < wd && j < wd && i >= j) Fm[(int64_t)(r0 + j) * ld + r0 + i] = blk[e];
    }
  }
  const int nb = (cmax + kTile - 1) / kTile;
  // Z <- B  (identity rows for pivots, L21 rows for the structure)
  for (int e = tid; e < nr * cmax; e += blockDim.x) {
    const int i = e % nr, c = e / nr, r = r0 + i;
    Zm[(int64_t)c * ld + r] = (r < npiv) ? (r == c ? 1.0 : 0.0) : Fm[(int64_t)c * ld + r];
  }
  __syncthreads();
  for (int cbi = nb - 1; cbi >= 0; --cbi) {
    const int cb = cbi * kTile;
    const int wb = min(kTile, npiv - cb);
#pragma unroll
    for (int e = tid; e < kTile * kTile; e += kZThreads) {
      const int i = e & 31, c = e >> 5;
      Ts[i][c] = (i < nr && c < wb) ? Zm[(int64_t)(cb + c) * ld + r0 + i] : 0.0;
      const int cp = e & 31;
      Ls[cp][c] = (cp < wb && c < wb && cp > c && !pair_skip(F.pivtype, cp, c))
                      ? ds[(int64_t)cbi * kTile * kTile + cp * kTile + c] : 0.0;
    }
    __syncthreads();
    if (warp == 0) {   // z Lblk = t, right to left, row in registers (independent FMAs)
      double z[kTile];
#pragma unroll
      for (int c = 0; c < kTile; ++c) z[c] = Ts[lane][c];
#pragma unroll
      for (int c = kTile - 1; c > 0; --c) {
#pragma unroll
        for (int cc = 0; cc < c; ++cc) z[cc] -= z[c] * Ls[c][cc];
      }
#pragma unroll
      for (int c = 0; c < kTile; ++c) Ts[lane][c] = z[c];
    }
    __syncthreads();
    for (int e = tid; e < kTile * kTile; e += blockDim.x) {
      const int i = e & 31, c = e >> 5;
      if (i < nr && c < wb) Zm[(int64_t)(cb + c) * ld + r0 + i] = Ts[i][c];
    }
    // right-looking update of the remaining column blocks: Z[:, blk] -= Zblk * L11[cb.., blk]
    for (int blk = warp; blk < cbi; blk += 8) {
      const int c0 = blk * kTile;
      double Bf[8][4];   // B fragments: L11[cb + kk + q][c0 + nf*8 + g]
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
#pragma unroll
        for (int nf = 0; nf < 4; ++nf) {
          const int kk = ks * 4 + q;
          Bf[ks][nf] = (kk < wb) ? Fm[(int64_t)(c0 + nf * 8 + g) * ld + cb + kk] : 0.0;
        }
      double acc[4][4][2];
#pragma unroll
      for (int mf = 0; mf < 4; ++mf)
#pragma unroll
        for (int nf = 0; nf < 4; ++nf) acc[mf][nf][0] = acc[mf][nf][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
        for (int mf = 0; mf < 4; ++mf) {
          const double a = Ts[mf * 8 + g][ks * 4 + q];
#pragma unroll
          for (int nf = 0; nf < 4; ++nf) dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], a, Bf[ks][nf]);
        }
      }
#pragma unroll
      for (int mf = 0; mf < 4; ++mf)
#pragma unroll
        for (int nf = 0; nf < 4; ++nf)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = mf * 8 + g, j = nf * 8 + 2 * q + h;
            if (i < nr) Zm[(int64_t)(c0 + j) * ld + r0 + i] -= acc[mf][nf][h];
          }
    }
    __syncthreads();
  }
}

// Forward solve, gather step (one CTA per front): v = [b(pivots); 0] + children updates
// (extend-add in fixed child order; rel maps are injective within a child).
__global__ void __launch_bounds__(kSolveThreads)
k_fwd_gather(const Work* __restrict__ work, const DFront* __restrict__ fronts,
             const int32_t* __restrict__ children, const int32_t* __restrict__ rel,
             const double* __restrict__ bperm, int64_t n, const double* __restrict__ ubuf,
             int64_t ustride, double* __restrict__ vbuf, int64_t vstride, int leading) {
  const int b = blockIdx.y;
  const DFront F = fronts[work[blockIdx.x].f];
  if (leading && F.is_root_p) return;
  const int tid = threadIdx.x;
  double* v = vbuf + (int64_t)b * vstride + F.voff;
  const double* bb = bperm + (int64_t)b * n;
  for (int i = tid; i < F.nrow; i += blockDim.x) v[i] = (i < F.npiv) ? bb[F.first + i] : 0.0;
  __syncthreads();
  for (int ci = F.child_begin; ci < F.child_end; ++ci) {
    const DFront C = fronts[children[ci]];
    const int cn = C.nrow - C.npiv;
    const double* uc = ubuf + (int64_t)b * ustride + C.uoff;
    const int32_t* rc = rel + C.rel_off;
    for (int t = tid; t < cn; t += blockDim.x) v[rc[t]] += uc[t];
    __syncthreads();
  }
}

// last-arriving CTA of a chunk group (ticket); partials are then summed in chunk order
__device__ __forceinline__ bool group_last(int* ticket, int nch) {
  __shared__ int last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(ticket, 1);
    last = (old == nch - 1);
    if (last) *ticket = 0;     // reset for the next solve
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// Forward solve, GEMV step on (front, 32-row tile, 64-column chunk):
//   partial_k = Z[rows, chunk] v[chunk]; the group's last CTA sums the chunks in order:
//   pivot rows -> z = D^{-1} y1 (zbuf); structure rows -> u = v2 - t (parent update).
__global__ void __launch_bounds__(kSolveThreads)
k_fwd(const Work* __restrict__ work, const DFront* __restrict__ fronts,
      const double* __restrict__ fstore, int64_t fstride, const double* __restrict__ zstore,
      int64_t zstride, const double* __restrict__ vbuf, int64_t vstride,
      double* __restrict__ zbuf, int64_t n, double* __restrict__ ubuf, int64_t ustride,
      double* __restrict__ part, int64_t pstride, int* __restrict__ tickets, int64_t n_groups,
      const int32_t* __restrict__ grp_nchunk, const int64_t* __restrict__ grp_base, int leading) {
  __shared__ double red[8][33];
  const int b = blockIdx.y;
  const Work wk = work[blockIdx.x];
  const DFront F = fronts[wk.f];
  if (leading && F.is_root_p) return;
  const int r0 = wk.a, k = wk.b, g = wk.c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(sgn::kFwdRows, F.nrow - r0);
  const int npiv = F.npiv;
  const int cend = (r0 < npiv) ? min(npiv, r0 + nr) : npiv;
  const int c_lo = k * sgn::kFwdCols, c_hi = min(c_lo + sgn::kFwdCols, cend);
  const double* Zm = zstore + (int64_t)b * zstride + F.zoff;
  const double* v = vbuf + (int64_t)b * vstride + F.voff;
  const int64_t ld = F.nrow;
  __shared__ double vs[sgn::kFwdCols];
  if (tid < c_hi - c_lo) vs[tid] = v[c_lo + tid];
  __syncthreads();
  double a0 = 0.0, a1 = 0.0;
  if (lane < nr) {
    const double* zr = Zm + r0 + lane;
    int c = c_lo + warp;
    for (; c + 8 < c_hi; c += 16) {
      a0 += zr[(int64_t)c * ld] * vs[c - c_lo];
      a1 += zr[(int64_t)(c + 8) * ld] * vs[c + 8 - c_lo];
    }
    if (c < c_hi) a0 += zr[(int64_t)c * ld] * vs[c - c_lo];
  }
  red[warp][lane] = a0 + a1;
  __syncthreads();
  const int nch = grp_nchunk[g];
  double* pp = part + (int64_t)b * pstride + grp_base[g];
  if (nch > 1) {
    if (warp == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w][lane];
      pp[k * 32 + lane] = t;
    }
    if (!group_last(tickets + (int64_t)b * n_groups + g, nch)) return;
  }
  if (warp != 0) return;
  double t = 0.0;
  if (nch > 1) {
    for (int kk = 0; kk < nch; ++kk) t += __ldcg(pp + kk * 32 + lane);
  } else {
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
  }
  const double tp = __shfl_xor_sync(0xffffffffu, t, 1);   // 2x2 pivot partner row
  if (lane >= nr) return;
  const int r = r0 + lane;
  if (r < npiv) {
    const double* Fm = fstore + (int64_t)b * fstride + F.foff;
    double* zb = zbuf + (int64_t)b * n;
    if (F.pivtype == 2) {
      const int re = r & ~1;
      const double a = Fm[(int64_t)re * ld + re], bq = Fm[(int64_t)re * ld + re + 1],
                   c = Fm[(int64_t)(re + 1) * ld + re + 1];
      const double det = a * c - bq * bq;
      zb[F.first + r] = ((r & 1) == 0) ? (c * t - bq * tp) / det : (a * t - bq * tp) / det;
    } else {
      zb[F.first + r] = t / Fm[(int64_t)r * ld + r];
    }
  } else {
    ubuf[(int64_t)b * ustride + F.uoff + (r - npiv)] = v[r] - t;
  }
}

// Backward solve on (front, 32-column tile, 256-row chunk): x1 = Z^T [z1; -x2] as column
// dots (warp per column, coalesced), chunk partials combined by the group's last CTA.
__global__ void __launch_bounds__(kSolveThreads)
k_bwd(const Work* __restrict__ work, const DFront* __restrict__ fronts,
      const int64_t* __restrict__ srows, const double* __restrict__ zstore, int64_t zstride,
      const double* __restrict__ zbuf, double* __restrict__ xbuf, int64_t n,
      double* __restrict__ part, int64_t pstride, int* __restrict__ tickets, int64_t n_groups,
      const int32_t* __restrict__ grp_nchunk, const int64_t* __restrict__ grp_base, int leading) {
  __shared__ double colsum[32];
  const int b = blockIdx.y;
  const Work wk = work[blockIdx.x];
  const DFront F = fronts[wk.f];
  const int c0 = wk.a, rs = wk.b, g = wk.c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int ncol = min(sgn::kBwdCols, F.npiv - c0);
  double* xb = xbuf + (int64_t)b * n;
  if (leading && F.is_root_p) {
    if (rs <= c0) for (int j = tid; j < ncol; j += blockDim.x) xb[F.first + c0 + j] = 0.0;
    return;
  }
  __shared__ double vs[sgn::kBwdRows];
  const double* zb = zbuf + (int64_t)b * n;
  const double* Zm = zstore + (int64_t)b * zstride + F.zoff;
  const int64_t ld = F.nrow;
  const int64_t* sr = srows + F.srow_off;
  const int np = F.npiv;
  const int re = min(rs + sgn::kBwdRows, F.nrow);
  for (int i = tid; i < re - rs; i += blockDim.x) {
    const int r = rs + i;
    vs[i] = (r < np) ? zb[F.first + r] : -xb[sr[r - np]];
  }
  __syncthreads();
  // warp w owns columns w, w+8, w+16, w+24 of the tile; all four dots advance together
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const double* col[4];
  int rbeg[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int j = c0 + warp + 8 * m;
    col[m] = Zm + (int64_t)j * ld;
    rbeg[m] = (warp + 8 * m < ncol) ? max(rs, j) : re;   // empty range for missing columns
  }
  for (int r = rs + lane; r < re; r += 32) {
    const double v = vs[r - rs];
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (r >= rbeg[m]) acc[m] += col[m][r] * v;
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    double a = acc[m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) colsum[warp + 8 * m] = a;
  }
  __syncthreads();
  const int nch = grp_nchunk[g];
  double* pp = part + (int64_t)b * pstride + grp_base[g];
  const int k = (rs - (c0 / sgn::kBwdRows) * sgn::kBwdRows) / sgn::kBwdRows;
  if (nch > 1) {
    if (tid < 32) pp[k * 32 + tid] = colsum[tid];
    if (!group_last(tickets + (int64_t)b * n_groups + g, nch)) return;
    if (tid < ncol) {
      double t = 0.0;
      for (int kk = 0; kk < nch; ++kk) t += __ldcg(pp + kk * 32 + tid);
      xb[F.first + c0 + tid] = t;
    }
  } else if (tid < ncol) {
    xb[F.first + c0 + tid] = colsum[tid];
  }
}

__global__ void k_permute_in(const double* __restrict__ x, double* __restrict__ y,
                             const int64_t* __restrict__ perm, int64_t n) {
  const int b = blockIdx.y;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    y[(int64_t)b * n + q] = x[(int64_t)b * n + perm[q]];
}
__global__ void k_permute_out(const double* __restrict__ y, double* __restrict__ x,
                              const int64_t* __restrict__ perm, int64_t n) {
  const int b = blockIdx.y;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
    x[(int64_t)b * n + perm[q]] = y[(int64_t)b * n + q];
}

// ------------------------------------------------------------------------------------
// Persistent dependency-driven triangular solve: ONE launch per solve.  Resident CTAs grab
// tasks (gather / forward GEMV / backward dots, see symbolic.cpp "persistent solve DAG") in
// topological order from a global head counter, spin on their (counter, target) waits with
// gpu-scope acquire loads, run the body and release their counter.  Every value produced
// inside the launch (v, u, z, x, chunk partials) is read with ld.global.cg (L2), never
// through a possibly stale L1 line.  The permutation in/out is folded into the gather
// (b[perm]) and the backward step (x[perm] = ...).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct SolveArgs {
  const sgn::Task* tasks; const int32_t* waits; int64_t ntask; int batch;
  int* head; int* cnt; int n_cnt;
  const DFront* fronts; const int64_t* srows; const int64_t* gptr; const int32_t* gsrc;
  const int64_t* perm; const double* fstore; int64_t fstride; const double* zstore; int64_t zstride;
  double* ubuf; int64_t ustride; double* zbuf; double* xbuf;
  int64_t n; double* part; int64_t pstride; int* tickets; int64_t n_groups;
  const int32_t* grp_nchunk; const int64_t* grp_base;
  const double* b_in; double* x_out; int leading; int nop; int mode;
  unsigned long long* trace;   // optional, 6 words per task: start, smid|signalled, prefetched, ready, combined, end
};

// thread 0 spins on the task's (counter, target) pairs; the CTA leaves together
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


__device__ __forceinline__ void dag_mark(const SolveArgs& A, int64_t idx, int slot) {
  if (A.trace && threadIdx.x == 0) A.trace[idx * 6 + slot] = gtimer();
}

__device__ __forceinline__ void dag_wait(const SolveArgs& A, const sgn::Task& T, const int* cnt) {
  if (threadIdx.x == 0) {
    for (int w = T.w0; w < T.w1; ++w) {
      const int* c = cnt + A.waits[2 * w];
      const int target = A.waits[2 * w + 1];
      if (A.mode & 1) { while (ld_acquire(c) < target) { } }
      else { while (ld_acquire(c) < target) __nanosleep(20); }
    }
  }
  __syncthreads();
}

// last-arriving CTA of a chunk group: one acq_rel ticket atomic (releases this CTA's
// partial, acquires the others'); the ticket is reset for the next solve
__device__ __forceinline__ bool dag_group_last(int* ticket, int nch) {
  __shared__ int last;
  __syncthreads();                   // the CTA's partial stores precede thread 0's release
  if (threadIdx.x == 0) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
    last = (old == nch - 1);
    if (last) *ticket = 0;
  }
  __syncthreads();
  return last != 0;
}

// deterministic sum of nch 32-wide chunk partials: warp w adds chunks w, w+8, ... (loads
// in flight together), warp 0 then adds the 8 warp sums in order.  Valid in warp 0.
__device__ __forceinline__ double dag_combine(const double* pp, int nch, double (*red)[33]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double t = 0.0;
#pragma unroll 4
  for (int kk = w; kk < nch; kk += 8) t += __ldcg(pp + kk * 32 + lane);
  red[w][lane] = t;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q][lane];
  }
  return s;
}

// Forward GEMV task (front, 32-row tile, 64-column chunk).  Before waiting it prefetches
// its Z tile (8 values per thread) and the inverse gather map of the v entries it needs
// (64 chunk columns + its own struct rows); after the children are done it forms those v
// entries (b + children updates in child order), multiplies, and the group's last CTA
// emits z = D^{-1} y1 (pivot rows) or u = v2 - t (struct rows, the parent's update).
__device__ bool dag_fwd(const SolveArgs& A, const sgn::Task& T, int b, const int* cnt, int64_t idx) {
  __shared__ double red[8][33];
  __shared__ double vs[sgn::kFwdCols + sgn::kFwdRows];
  const DFront F = A.fronts[T.f];
  const int r0 = T.a, k = T.b, g = T.c;
  if (A.nop || (A.leading && F.is_root_p)) { dag_wait(A, T, cnt); return k == 0; }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nr = min(sgn::kFwdRows, F.nrow - r0);
  const int npiv = F.npiv;
  const int cend = (r0 < npiv) ? min(npiv, r0 + nr) : npiv;
  const int c_lo = k * sgn::kFwdCols, c_hi = min(c_lo + sgn::kFwdCols, cend);
  const double* Zm = A.zstore + (int64_t)b * A.zstride + F.zoff;
  const int64_t ld = F.nrow;
  double z[8];
  {
    const double* zr = Zm + r0 + lane;
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int c = c_lo + warp + 8 * m;
      z[m] = (lane < nr && c < c_hi) ? zr[(int64_t)c * ld] : 0.0;
    }
  }
  int vr = -1;
  if (tid < sgn::kFwdCols) {
    if (c_lo + tid < c_hi) vr = c_lo + tid;
  } else if (tid < sgn::kFwdCols + sgn::kFwdRows) {
    const int r = r0 + tid - sgn::kFwdCols;
    if (r < F.nrow && r >= npiv) vr = r;
  }
  double base = 0.0;
  int64_t q0 = 0, q1 = 0;
  int sq[4] = {0, 0, 0, 0};
  if (vr >= 0) {
    base = (vr < npiv) ? A.b_in[(int64_t)b * A.n + A.perm[F.first + vr]] : 0.0;
    q0 = A.gptr[F.voff + vr];
    q1 = A.gptr[F.voff + vr + 1];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (q0 + j < q1) sq[j] = A.gsrc[q0 + j];
  }
  // pivot rows of this tile: the D block entries the final step needs (static)
  double da = 1.0, db = 0.0, dc = 1.0;
  if (warp == 0 && lane < nr && r0 + lane < npiv) {
    const double* Fm = A.fstore + (int64_t)b * A.fstride + F.foff;
    const int r = r0 + lane;
    if (F.pivtype == 2) {
      const int re = r & ~1;
      da = Fm[(int64_t)re * ld + re]; db = Fm[(int64_t)re * ld + re + 1]; dc = Fm[(int64_t)(re + 1) * ld + re + 1];
    } else {
      da = Fm[(int64_t)r * ld + r];
    }
  }
  dag_mark(A, idx, 2);
  dag_wait(A, T, cnt);
  dag_mark(A, idx, 3);
  if (tid < sgn::kFwdCols + sgn::kFwdRows) {
    double v = 0.0;
    if (vr >= 0) {
      const double* ub = A.ubuf + (int64_t)b * A.ustride;
      double u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) u[j] = (q0 + j < q1) ? __ldcg(ub + sq[j]) : 0.0;
      v = base;
#pragma unroll
      for (int j = 0; j < 4; ++j) if (q0 + j < q1) v += u[j];
      for (int64_t q = q0 + 4; q < q1; ++q) v += __ldcg(ub + A.gsrc[q]);
    }
    vs[tid] = v;
  }
  __syncthreads();
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < 8; ++m) acc += z[m] * vs[warp + 8 * m];
  red[warp][lane] = acc;
  __syncthreads();
  const int nch = A.grp_nchunk[g];
  double t = 0.0;
  if (warp == 0) {
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
  }
  if (nch > 1) {
    double* pp = A.part + (int64_t)b * A.pstride + A.grp_base[g];
    if (warp == 0) pp[k * 32 + lane] = t;
    if (!dag_group_last(A.tickets + (int64_t)b * A.n_groups + g, nch)) return false;
    dag_mark(A, idx, 4);
    t = dag_combine(pp, nch, red);
  }
  if (warp == 0) {
    const double tp = __shfl_xor_sync(0xffffffffu, t, 1);   // 2x2 pivot partner row
    if (lane < nr) {
      const int r = r0 + lane;
      if (r < npiv) {
        double* zb = A.zbuf + (int64_t)b * A.n;
        if (F.pivtype == 2) {
          const double det = da * dc - db * db;
          zb[F.first + r] = ((r & 1) == 0) ? (dc * t - db * tp) / det : (da * t - db * tp) / det;
        } else {
          zb[F.first + r] = t / da;
        }
      } else {
        A.ubuf[(int64_t)b * A.ustride + F.uoff + (r - npiv)] = vs[sgn::kFwdCols + lane] - t;
      }
    }
  }
  return true;
}

// Backward task (front, 32-column tile, 128-row chunk): x1 = Z^T [z1; -x2] as column dots.
// Z (16 values per thread) and the struct-row map are prefetched before the wait.
__device__ bool dag_bwd(const SolveArgs& A, const sgn::Task& T, int b, const int* cnt, int64_t idx) {
  __shared__ double colsum[32];
  __shared__ double vs[sgn::kBwdRows];
  const DFront F = A.fronts[T.f];
  const int c0 = T.a, rs = T.b, g = T.c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncol = min(sgn::kBwdCols, F.npiv - c0);
  double* xb = A.xbuf + (int64_t)b * A.n;
  double* xo = A.x_out + (int64_t)b * A.n;
  const bool first_chunk = (rs == (c0 / sgn::kBwdRows) * sgn::kBwdRows);
  if (A.nop) { dag_wait(A, T, cnt); return first_chunk; }
  if (A.leading && F.is_root_p) {
    dag_wait(A, T, cnt);
    if (first_chunk)
      for (int j = tid; j < ncol; j += blockDim.x) {
        xb[F.first + c0 + j] = 0.0;
        xo[A.perm[F.first + c0 + j]] = 0.0;
      }
    return first_chunk;
  }
  const double* Zm = A.zstore + (int64_t)b * A.zstride + F.zoff;
  const int64_t ld = F.nrow;
  const int np = F.npiv;
  const int re = min(rs + sgn::kBwdRows, F.nrow);
  double z[4][4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int j = c0 + warp + 8 * m;
    const bool colok = (warp + 8 * m < ncol);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = rs + lane + 32 * i;
      z[m][i] = (colok && r < re && r >= j) ? Zm[(int64_t)j * ld + r] : 0.0;
    }
  }
  int64_t srow = -1;
  if (tid < re - rs && rs + tid >= np) srow = A.srows[F.srow_off + rs + tid - np];
  dag_mark(A, idx, 2);
  dag_wait(A, T, cnt);
  dag_mark(A, idx, 3);
  if (tid < sgn::kBwdRows) {
    double v = 0.0;
    if (tid < re - rs)
      v = (rs + tid < np) ? __ldcg(A.zbuf + (int64_t)b * A.n + F.first + rs + tid) : -__ldcg(xb + srow);
    vs[tid] = v;
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    double a = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) a += z[m][i] * vs[lane + 32 * i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) colsum[warp + 8 * m] = a;
  }
  __syncthreads();
  const int nch = A.grp_nchunk[g];
  double* pp = A.part + (int64_t)b * A.pstride + A.grp_base[g];
  const int k = (rs - (c0 / sgn::kBwdRows) * sgn::kBwdRows) / sgn::kBwdRows;
  double t = 0.0;
  if (nch > 1) {
    __shared__ double red[8][33];
    if (tid < 32) pp[k * 32 + tid] = colsum[tid];
    if (!dag_group_last(A.tickets + (int64_t)b * A.n_groups + g, nch)) return false;
    dag_mark(A, idx, 4);
    t = dag_combine(pp, nch, red);
  } else if (tid < ncol) {
    t = colsum[tid];
  }
  if (tid < ncol) {
    xb[F.first + c0 + tid] = t;
    xo[A.perm[F.first + c0 + tid]] = t;
  }
  return true;
}

__global__ void __launch_bounds__(kSolveThreads)
k_solve_dag(const SolveArgs A) {
  __shared__ int s_idx;
  const int64_t total = A.ntask * A.batch;
  for (;;) {
    __syncthreads();                               // s_idx of the previous task consumed
    if (threadIdx.x == 0) s_idx = atomicAdd(A.head, 1);
    __syncthreads();
    const int64_t idx = s_idx;
    if (idx >= total) return;
    const int64_t ti = idx / A.batch;
    const int b = (int)(idx - ti * A.batch);
    const sgn::Task T = A.tasks[ti];
    int* cnt = A.cnt + (int64_t)b * A.n_cnt;
    unsigned long long t0 = 0;
    if (A.trace && threadIdx.x == 0) t0 = gtimer();
    const bool sig = (T.kind == sgn::T_FWD) ? dag_fwd(A, T, b, cnt, idx) : dag_bwd(A, T, b, cnt, idx);
    __syncthreads();                               // every thread's writes precede the release
    if (sig && threadIdx.x == 0) {
      asm volatile("fence.acq_rel.gpu;\n\tred.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(cnt + T.sig) : "memory");
    }
    if (A.trace && threadIdx.x == 0) {
      unsigned long long* tr = A.trace + idx * 6;
      tr[0] = t0;
      tr[5] = gtimer();
      tr[1] = ((unsigned long long)smid() << 48) | (sig ? 1ull : 0ull);
    }
  }
}

// ------------------------------------------------------------------------------------
// SpMV on the symmetric pattern (CSC == CSR), 8 lanes per row
// ------------------------------------------------------------------------------------
__global__ void k_spmv(const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                       const double* __restrict__ vals, int64_t vstride,
                       const double* __restrict__ x, double* __restrict__ y, int64_t n,
                       int64_t p_lo, int64_t p_hi) {
  const int b = blockIdx.y;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3;
  const int sub = threadIdx.x & 7;
  const bool valid = row < n;
  const double* vb = vals + (int64_t)b * vstride;
  const double* xb = x + (int64_t)b * n;
  double acc = 0.0;
  const int64_t kb = valid ? ptr[row] : 0, ke = valid ? ptr[row + 1] : 0;
  for (int64_t k = kb + sub; k < ke; k += 8) {
    const int32_t c = idx[k];
    if (c >= p_lo && c < p_hi) continue;
    acc += vb[k] * xb[c];
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if (valid && sub == 0) y[(int64_t)b * n + row] = (row >= p_lo && row < p_hi) ? 0.0 : acc;
}

// ------------------------------------------------------------------------------------
// deterministic batched BLAS-1 for BiCGSTAB (fixed reduction trees)
// ------------------------------------------------------------------------------------
constexpr int kDotBlocks = 64;
constexpr int kDotThreads = 256;

// up to 2 dot products in one pass: out[b*2+0] = a.b, out[b*2+1] = c.d (if c)
__global__ void __launch_bounds__(kDotThreads)
k_dot_partial(const double* __restrict__ a, const double* __restrict__ bvec,
              const double* __restrict__ c, const double* __restrict__ d, int64_t n,
              double* __restrict__ partial) {
  __shared__ double s0[kDotThreads], s1[kDotThreads];
  const int b = blockIdx.y;
  const double* ab = a + (int64_t)b * n;
  const double* bb = bvec + (int64_t)b * n;
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    acc0 += ab[i] * bb[i];
    if (c) acc1 += c[(int64_t)b * n + i] * d[(int64_t)b * n + i];
  }
  s0[threadIdx.x] = acc0;
  s1[threadIdx.x] = acc1;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) { s0[threadIdx.x] += s0[threadIdx.x + s]; s1[threadIdx.x] += s1[threadIdx.x + s]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[((int64_t)b * kDotBlocks + blockIdx.x) * 2 + 0] = s0[0];
    partial[((int64_t)b * kDotBlocks + blockIdx.x) * 2 + 1] = s1[0];
  }
}

struct BiState {
  double rho, alpha, omega, bnorm, best_res, res, dot0, dot1;
  int32_t active, iters, reason, pad;
};

// reduce partials and run one scalar step of BiCGSTAB per instance.
// step: 0 = bnorm, 1 = initial residual (res0), 2 = rho, 3 = alpha, 4 = omega, 5 = residual
__global__ void k_dot_final(const double* __restrict__ partial, BiState* __restrict__ st,
                            int step, double tol, int32_t it) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  double s0 = 0.0, s1 = 0.0;
  for (int k = 0; k < kDotBlocks; ++k) {
    s0 += partial[((int64_t)b * kDotBlocks + k) * 2 + 0];
    s1 += partial[((int64_t)b * kDotBlocks + k) * 2 + 1];
  }
  BiState& S = st[b];
  S.dot0 = s0;
  S.dot1 = s1;
  if (step == 0) {
    S.bnorm = sqrt(s0);
    S.iters = 0; S.reason = 0; S.active = 1;
    S.rho = S.alpha = S.omega = 1.0;
    if (S.bnorm == 0.0) { S.active = 0; S.res = 0.0; S.best_res = 0.0; S.reason = 4; }
    return;
  }
  if (!S.active) return;
  if (step == 1) {
    S.res = sqrt(s0) / S.bnorm;
    S.best_res = S.res;
    if (S.res <= tol) { S.active = 0; S.reason = 1; }
  } else if (step == 2) {
    const double rho_new = s0;
    if (rho_new == 0.0 || S.omega == 0.0) { S.active = 0; S.reason = 2; S.iters = it - 1; return; }
    const double beta = (rho_new / S.rho) * (S.alpha / S.omega);
    S.rho = rho_new;
    S.dot1 = beta;
  } else if (step == 3) {
    if (s0 == 0.0) { S.active = 0; S.reason = 2; S.iters = it - 1; return; }
    S.alpha = S.rho / s0;
  } else if (step == 4) {
    // s0 = t.t, s1 = t.s
    S.omega = (s0 > 0.0) ? s1 / s0 : 0.0;
  } else if (step == 5) {
    S.res = sqrt(s0) / S.bnorm;
    S.iters = it;
    if (S.res < S.best_res) { S.best_res = S.res; S.reason = 10; /* copy best */ }
    if (S.res <= tol) { S.active = 0; S.reason = 1; }
  }
}

// vector kernels (each masked by the instance's active flag)
// mode 0: out = x + a*y          (a from st field)
__global__ void k_vec(int mode, const BiState* __restrict__ st, int64_t n,
                      double* __restrict__ o, const double* __restrict__ x,
                      const double* __restrict__ y, const double* __restrict__ z,
                      double* __restrict__ o2, double* __restrict__ o3) {
  const int b = blockIdx.y;
  const BiState S = st[b];
  if (mode != 9 && mode != 7 && !S.active) return;
  const int64_t base = (int64_t)b * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = base + i;
    switch (mode) {
      case 0:  // r = b - Ax ;  o = x - y
        o[k] = x[k] - y[k];
        break;
      case 1:  // p = r + beta (p - omega v)   beta in dot1 (set by step 2)
        o[k] = x[k] + S.dot1 * (o[k] - S.omega * y[k]);
        break;
      case 2:  // s = r - alpha v
        o[k] = x[k] - S.alpha * y[k];
        break;
      case 3:  // x += alpha p + omega s ; r = s - omega t   (o = x, x = p, y = s, z = t, o2 = r)
        o[k] += S.alpha * x[k] + S.omega * y[k];
        o2[k] = y[k] - S.omega * z[k];
        break;
      case 4:  // copy o = x
        o[k] = x[k];
        break;
      case 7:  // best-copy when step 5 flagged a new best iterate (reason 10)
        if (S.reason == 10) o[k] = x[k];
        break;
      case 9:  // unconditional copy
        o[k] = x[k];
        break;
    }
  }
}

__global__ void k_clear_reason(BiState* st) {
  const int b = blockIdx.x;
  if (threadIdx.x == 0 && st[b].reason == 10) st[b].reason = 0;
}

// final select: out = (converged at last iterate) ? x : best
__global__ void k_select(const BiState* __restrict__ st, int64_t n, const double* __restrict__ x,
                         const double* __restrict__ best, double* __restrict__ out) {
  const int b = blockIdx.y;
  const BiState S = st[b];
  const int64_t base = (int64_t)b * n;
  const bool use_x = (S.reason == 1) || (S.reason == 4);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[base + i] = (S.reason == 4) ? 0.0 : (use_x ? x[base + i] : best[base + i]);
}

// ------------------------------------------------------------------------------------
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  int alloc(size_t cnt) {
    n = cnt;
    if (cnt == 0) return 0;
    cudaError_t e = cudaMalloc(&p, cnt * sizeof(T));
    if (e != cudaSuccess) { sgn::last_error() = std::string("cudaMalloc: ") + cudaGetErrorString(e); return SGN_CUDA_ERROR; }
    return 0;
  }
  int upload(const std::vector<T>& v) {
    int rc = alloc(v.size());
    if (rc) return rc;
    if (!v.empty()) {
      cudaError_t e = cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) { sgn::last_error() = std::string("cudaMemcpy: ") + cudaGetErrorString(e); return SGN_CUDA_ERROR; }
    }
    return 0;
  }
};

}  // namespace

struct sgn_symbolic_s {
  sgn::Symbolic s;
};

struct sgn_factor_s {
  sgn_symbolic sym = nullptr;
  int32_t batch = 1;
  int64_t n = 0;
  DevBuf<DFront> fronts;
  DevBuf<int32_t> children, rel, tile_loc, lvl_fronts, idx32;
  DevBuf<int64_t> srows, perm, tile_ptr, tile_nnz, indptr;
  DevBuf<int8_t> kind_pos;
  DevBuf<Work> work;
  DevBuf<double> fstore, wstore, ubuf, vbuf, y, zstore, zbuf, xbuf, part, dscr;
  DevBuf<int> tickets;
  DevBuf<int32_t> grp_nchunk;
  DevBuf<int64_t> grp_base;
  DevBuf<long long> status;
  DevBuf<sgn::Task> stasks;
  DevBuf<int32_t> swaits, gsrc;
  DevBuf<int64_t> gptr;
  DevBuf<int64_t> trace;        // SGN_DAG_TRACE=1: 3 words per solve task (diagnostics)
  DevBuf<int> scnt;             // [head | batch x n_scnt counters], zeroed before every solve
  int solve_grid = 0;
  std::vector<int64_t> lvl_off;  // level -> offset into lvl_fronts
  // BiCGSTAB workspace
  DevBuf<double> bx, br, brh, bp, bv, bs, bt, btmp, bbest, bb, bscr, partial;
  DevBuf<BiState> bst;
  bool bicg_ready = false;
  // captured triangular-solve graphs (index = flags)
  struct SolveGraph {
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t in_node = nullptr, out_node = nullptr;
    cudaKernelNodeParams in_p{}, out_p{};
    int64_t kernels = 0;
  } graphs[2];
  std::vector<cudaGraph_t> graph_templates;
  DevBuf<double> gin, gout;   // placeholder endpoints used only while capturing
  const double* bbuf_in() { if (!gin.p) gin.alloc((size_t)batch * std::max<int64_t>(n, 1)); return gin.p; }
  double* bbuf_out() { if (!gout.p) gout.alloc((size_t)batch * std::max<int64_t>(n, 1)); return gout.p; }
  ~sgn_factor_s() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto g : graph_templates) cudaGraphDestroy(g);
  }
};

namespace {

int launch_solve_raw(sgn_factor f, const double* d_b, double* d_x, int32_t flags, cudaStream_t st) {
  const sgn::Symbolic& s = f->sym->s;
  const int64_t n = s.n;
  if (n == 0) return SGN_OK;
  const dim3 pg((unsigned)std::min<int64_t>((n + 255) / 256, 1024), f->batch);
  sgn::count_launch();
  k_permute_in<<<pg, 256, 0, st>>>(d_b, f->y.p, f->perm.p, n);
  const int leading = (flags & SGN_SOLVE_LEADING) ? 1 : 0;
  for (int32_t lv = 0; lv < s.n_levels; ++lv) {
    if (s.gat_cnt[lv]) {
      sgn::count_launch();
      k_fwd_gather<<<dim3((unsigned)s.gat_cnt[lv], f->batch), kSolveThreads, 0, st>>>(
          f->work.p + s.gat_off[lv], f->fronts.p, f->children.p, f->rel.p, f->y.p, n, f->ubuf.p,
          s.u_doubles, f->vbuf.p, s.v_doubles, leading);
    }
    if (s.fwd_cnt[lv]) {
      sgn::count_launch();
      k_fwd<<<dim3((unsigned)s.fwd_cnt[lv], f->batch), kSolveThreads, 0, st>>>(
          f->work.p + s.fwd_off[lv], f->fronts.p, f->fstore.p, s.front_doubles, f->zstore.p,
          s.z_doubles, f->vbuf.p, s.v_doubles, f->zbuf.p, n, f->ubuf.p, s.u_doubles, f->part.p,
          s.part_doubles, f->tickets.p, s.n_groups, f->grp_nchunk.p, f->grp_base.p, leading);
    }
  }
  for (int32_t lv = s.n_levels - 1; lv >= 0; --lv) {
    if (!s.bwd_cnt[lv]) continue;
    sgn::count_launch();
    k_bwd<<<dim3((unsigned)s.bwd_cnt[lv], f->batch), kSolveThreads, 0, st>>>(
        f->work.p + s.bwd_off[lv], f->fronts.p, f->srows.p, f->zstore.p, s.z_doubles, f->zbuf.p,
        f->xbuf.p, n, f->part.p, s.part_doubles, f->tickets.p, s.n_groups, f->grp_nchunk.p,
        f->grp_base.p, leading);
  }
  sgn::count_launch();
  k_permute_out<<<pg, 256, 0, st>>>(f->xbuf.p, d_x, f->perm.p, n);
  CUDA_TRY(cudaGetLastError());
  return SGN_OK;
}


// One solve = a counter reset + ONE persistent dependency-driven launch (k_solve_dag).
int launch_solve_dag(sgn_factor f, const double* d_b, double* d_x, int32_t flags, cudaStream_t st) {
  const sgn::Symbolic& s = f->sym->s;
  SolveArgs A;
  A.tasks = f->stasks.p; A.waits = f->swaits.p; A.ntask = (int64_t)s.stasks.size(); A.batch = f->batch;
  A.head = f->scnt.p; A.cnt = f->scnt.p + 1; A.n_cnt = s.n_scnt;
  A.fronts = f->fronts.p; A.srows = f->srows.p; A.gptr = f->gptr.p; A.gsrc = f->gsrc.p;
  A.perm = f->perm.p; A.fstore = f->fstore.p; A.fstride = s.front_doubles;
  A.zstore = f->zstore.p; A.zstride = s.z_doubles; A.ubuf = f->ubuf.p; A.ustride = s.u_doubles;
  A.zbuf = f->zbuf.p; A.xbuf = f->xbuf.p; A.n = s.n;
  A.part = f->part.p; A.pstride = s.part_doubles; A.tickets = f->tickets.p; A.n_groups = s.n_groups;
  A.grp_nchunk = f->grp_nchunk.p; A.grp_base = f->grp_base.p;
  A.b_in = d_b; A.x_out = d_x; A.leading = (flags & SGN_SOLVE_LEADING) ? 1 : 0;
  { const char* e = getenv("SGN_DAG_NOP"); A.nop = (e && *e == '1') ? 1 : 0; }
  A.trace = nullptr;   // SGN_DAG_TRACE=1: 6 words per task
  { const char* e = getenv("SGN_DAG_MODE"); A.mode = e ? atoi(e) : 0; }
  { const char* e = getenv("SGN_DAG_TRACE");
    if (e && *e == '1') {
      if (!f->trace.p && f->trace.alloc((size_t)6 * std::max<int64_t>(1, (int64_t)s.stasks.size() * f->batch))) return SGN_CUDA_ERROR;
      A.trace = (unsigned long long*)f->trace.p;
      CUDA_TRY(cudaMemsetAsync(f->trace.p, 0, f->trace.n * sizeof(int64_t), st));
    } }
  CUDA_TRY(cudaMemsetAsync(f->scnt.p, 0, f->scnt.n * sizeof(int), st));
  const int64_t total = A.ntask * A.batch;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(f->solve_grid, total));
  sgn::count_launch();
  k_solve_dag<<<grid, kSolveThreads, 0, st>>>(A);
  CUDA_TRY(cudaGetLastError());
  return SGN_OK;
}

static bool use_level_solve() {
  static const int v = [] { const char* e = getenv("SGN_SOLVE_LEVELS"); return (e && *e == '1') ? 1 : 0; }();
  return v != 0;
}

// Level-scheduled alternative (SGN_SOLVE_LEVELS=1, kept for A/B timing): a fixed launch
// sequence per (factor, flags), captured once as a CUDA graph and replayed, patching only
// the permute-in / permute-out pointer arguments.
int launch_solve(sgn_factor f, const double* d_b, double* d_x, int32_t flags, cudaStream_t st) {
  const int64_t n = f->n;
  if (n == 0) return SGN_OK;
  if (!use_level_solve()) return launch_solve_dag(f, d_b, d_x, flags, st);
  auto& G = f->graphs[(flags & SGN_SOLVE_LEADING) ? 1 : 0];
  if (!G.exec) {
    const double* cap_in = f->bbuf_in();   // allocate before capturing
    double* cap_out = f->bbuf_out();
    if (!cap_in || !cap_out) { sgn::last_error() = "graph placeholder allocation failed"; return SGN_CUDA_ERROR; }
    CUDA_TRY(cudaDeviceSynchronize());
    cudaStream_t cs;
    CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph;
    CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    const int64_t before = sgn::launch_count();
    int rc = launch_solve_raw(f, cap_in, cap_out, flags, cs);
    sgn::count_launch(before - sgn::launch_count());   // captured, not launched
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (rc) return rc;
    if (e != cudaSuccess) { sgn::last_error() = std::string("capture: ") + cudaGetErrorString(e); return SGN_CUDA_ERROR; }
    size_t nn = 0;
    CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CUDA_TRY(cudaGraphGetNodes(graph, nodes.data(), &nn));
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      CUDA_TRY(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      ++G.kernels;
      cudaKernelNodeParams p;
      CUDA_TRY(cudaGraphKernelNodeGetParams(nd, &p));
      if (p.func == (void*)k_permute_in) { G.in_node = nd; G.in_p = p; }
      if (p.func == (void*)k_permute_out) { G.out_node = nd; G.out_p = p; }
    }
    CUDA_TRY(cudaGraphInstantiate(&G.exec, graph, 0));
    // the instantiated exec keeps its own copy; node handles stay valid for SetParams
    G.in_node = G.in_node; G.out_node = G.out_node;
    f->graph_templates.push_back(graph);
  }
  const double* b_arg = d_b;
  double* y_arg = f->y.p;
  const int64_t* perm_arg = f->perm.p;
  int64_t n_arg = n;
  void* in_args[] = {(void*)&b_arg, (void*)&y_arg, (void*)&perm_arg, (void*)&n_arg};
  cudaKernelNodeParams pin = G.in_p;
  pin.kernelParams = in_args;
  pin.extra = nullptr;
  CUDA_TRY(cudaGraphExecKernelNodeSetParams(G.exec, G.in_node, &pin));
  const double* xs_arg = f->xbuf.p;
  double* x_arg = d_x;
  void* out_args[] = {(void*)&xs_arg, (void*)&x_arg, (void*)&perm_arg, (void*)&n_arg};
  cudaKernelNodeParams pout = G.out_p;
  pout.kernelParams = out_args;
  pout.extra = nullptr;
  CUDA_TRY(cudaGraphExecKernelNodeSetParams(G.exec, G.out_node, &pout));
  CUDA_TRY(cudaGraphLaunch(G.exec, st));
  sgn::count_launch(G.kernels);
  return SGN_OK;
}

int launch_spmv(sgn_factor f, const double* vals, int64_t vstride, const double* x, double* y,
                int32_t flags, cudaStream_t st) {
  const sgn::Symbolic& s = f->sym->s;
  const int64_t n = s.n;
  if (n == 0) return SGN_OK;
  int64_t p_lo = 0, p_hi = 0;
  if ((flags & SGN_SOLVE_LEADING) && s.pair_mode) { p_lo = s.n_x; p_hi = s.n_x + s.n_p; }
  const int64_t threads = n * 8;
  sgn::count_launch();
  k_spmv<<<dim3((unsigned)((threads + 255) / 256), f->batch), 256, 0, st>>>(
      f->indptr.p, f->idx32.p, vals, vstride, x, y, n, p_lo, p_hi);
  CUDA_TRY(cudaGetLastError());
  return SGN_OK;
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

const char* sgn_last_error(void) { return sgn::last_error().c_str(); }
int sgn_version(void) { return 1; }
int64_t sgn_launch_count(void) { return sgn::launch_count(); }

int sgn_device_sync(void* stream) {
  CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return SGN_OK;
}

int sgn_symbolic_create(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t n_x,
                        int64_t n_p, int64_t n_c, int32_t leaf_size, sgn_symbolic* out,
                        int64_t* pivot_index) {
  try {
    if (!out || !indptr || n < 0) { sgn::last_error() = "bad arguments"; return SGN_INVALID; }
    auto h = std::make_unique<sgn_symbolic_s>();
    h->s.n = n; h->s.n_x = n_x; h->s.n_p = n_p; h->s.n_c = n_c;
    h->s.indptr.assign(indptr, indptr + n + 1);
    const int64_t nnz = h->s.indptr[n];
    h->s.indices.assign(indices, indices + nnz);
    int64_t piv = -1;
    int rc = sgn::build_symbolic(h->s, leaf_size, &piv);
    if (pivot_index) *pivot_index = piv;
    if (rc) return rc;
    *out = h.release();
    return SGN_OK;
  } catch (const std::exception& e) {
    sgn::last_error() = e.what();
    return SGN_INVALID;
  }
}

int sgn_symbolic_get_stats(sgn_symbolic h, sgn_symbolic_stats* o) {
  const sgn::Symbolic& s = h->s;
  o->n = s.n;
  o->n_fronts = (int64_t)s.fronts.size();
  o->n_levels = s.n_levels;
  o->nnz_l = s.nnz_l;
  o->front_doubles = s.front_doubles;
  o->max_front = s.max_front;
  o->max_piv = s.max_piv;
  o->launches = (int64_t)s.launches.size();
  o->flops = s.flops;
  o->pair_mode = s.pair_mode ? 1 : 0;
  return SGN_OK;
}

int sgn_symbolic_get_perm(sgn_symbolic h, int64_t* perm) {
  std::copy(h->s.perm.begin(), h->s.perm.end(), perm);
  return SGN_OK;
}

int sgn_symbolic_get_fronts(sgn_symbolic h, int64_t* first, int64_t* npiv, int64_t* nrow,
                            int64_t* parent, int64_t* rows_ptr, int64_t* rows) {
  const sgn::Symbolic& s = h->s;
  int64_t at = 0;
  for (size_t k = 0; k < s.fronts.size(); ++k) {
    const sgn::Front& F = s.fronts[k];
    if (first) first[k] = F.first;
    if (npiv) npiv[k] = F.npiv;
    if (nrow) nrow[k] = F.nrow;
    if (parent) parent[k] = F.parent;
    if (rows_ptr) rows_ptr[k] = at;
    for (int32_t i = 0; i < F.nrow; ++i) {
      if (rows) rows[at] = (i < F.npiv) ? F.first + i : s.srows[F.srow_off + i - F.npiv];
      ++at;
    }
  }
  if (rows_ptr) rows_ptr[s.fronts.size()] = at;
  return SGN_OK;
}

void sgn_symbolic_destroy(sgn_symbolic h) { delete h; }

int sgn_factor_create(sgn_symbolic h, int32_t batch, sgn_factor* out) {
  if (!h || batch < 1 || !out) { sgn::last_error() = "bad arguments"; return SGN_INVALID; }
  auto f = std::make_unique<sgn_factor_s>();
  f->sym = h;
  f->batch = batch;
  const sgn::Symbolic& s = h->s;
  f->n = s.n;
  std::vector<DFront> df(s.fronts.size());
  for (size_t k = 0; k < s.fronts.size(); ++k) {
    const sgn::Front& F = s.fronts[k];
    DFront& d = df[k];
    d.first = F.first; d.foff = F.foff; d.srow_off = F.srow_off; d.rel_off = F.rel_off;
    d.uoff = F.uoff; d.woff = F.woff; d.voff = F.voff; d.tile_base = F.tile_base;
    d.zoff = F.zoff; d.doff = F.doff;
    d.npiv = F.npiv; d.nrow = F.nrow; d.parent = F.parent; d.pivtype = F.pivtype;
    d.child_begin = F.child_begin; d.child_end = F.child_end; d.is_root_p = F.is_root_p;
    d.level = F.level;
  }
  std::vector<int32_t> lf;
  f->lvl_off.assign(s.n_levels + 1, 0);
  for (int32_t lv = 0; lv < s.n_levels; ++lv) {
    f->lvl_off[lv] = (int64_t)lf.size();
    lf.insert(lf.end(), s.level_fronts[lv].begin(), s.level_fronts[lv].end());
  }
  f->lvl_off[s.n_levels] = (int64_t)lf.size();
  std::vector<int32_t> idx32(s.indices.begin(), s.indices.end());
  int rc = 0;
  if ((rc = f->fronts.upload(df)) || (rc = f->children.upload(s.children)) ||
      (rc = f->rel.upload(s.rel)) || (rc = f->tile_loc.upload(s.tile_loc)) ||
      (rc = f->lvl_fronts.upload(lf)) || (rc = f->idx32.upload(idx32)) ||
      (rc = f->srows.upload(s.srows)) || (rc = f->perm.upload(s.perm)) ||
      (rc = f->tile_ptr.upload(s.tile_ptr)) || (rc = f->tile_nnz.upload(s.tile_nnz)) ||
      (rc = f->indptr.upload(s.indptr)) || (rc = f->kind_pos.upload(s.kind_pos)) ||
      (rc = f->work.upload(s.work)))
    return rc;
  const size_t B = (size_t)batch;
  if ((rc = f->fstore.alloc(B * std::max<int64_t>(s.front_doubles, 1))) ||
      (rc = f->wstore.alloc(B * std::max<int64_t>(s.w_doubles, 1))) ||
      (rc = f->ubuf.alloc(B * std::max<int64_t>(s.u_doubles, 1))) ||
      (rc = f->vbuf.alloc(B * std::max<int64_t>(s.v_doubles, 1))) ||
      (rc = f->y.alloc(B * std::max<int64_t>(s.n, 1))) || (rc = f->status.alloc(B)) ||
      (rc = f->zstore.alloc(B * std::max<int64_t>(s.z_doubles, 1))) ||
      (rc = f->zbuf.alloc(B * std::max<int64_t>(s.n, 1))) ||
      (rc = f->xbuf.alloc(B * std::max<int64_t>(s.n, 1))))
    return rc;
  if ((rc = f->part.alloc(B * std::max<int64_t>(s.part_doubles, 1))) ||
      (rc = f->dscr.alloc(B * std::max<int64_t>(s.d_doubles, 1))) ||
      (rc = f->tickets.alloc(B * std::max<int64_t>(s.n_groups, 1))) ||
      (rc = f->grp_nchunk.upload(s.grp_nchunk)) || (rc = f->grp_base.upload(s.grp_base)) ||
      (rc = f->stasks.upload(s.stasks)) || (rc = f->swaits.upload(s.swaits)) ||
      (rc = f->gptr.upload(s.gptr)) || (rc = f->gsrc.upload(s.gsrc)) ||
      (rc = f->scnt.alloc(1 + B * std::max<int64_t>(s.n_scnt, 1))))
    return rc;
  {
    int dev = 0, sms = 0, per_sm = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve_dag, kSolveThreads, 0));
    f->solve_grid = std::max(1, sms * std::max(per_sm, 1));
  }
  CUDA_TRY(cudaMemset(f->tickets.p, 0, f->tickets.n * sizeof(int)));
  // Z11 = L11^{-1} is lower triangular: the strictly upper part stays zero forever
  CUDA_TRY(cudaMemset(f->zstore.p, 0, f->zstore.n * sizeof(double)));
  *out = f.release();
  return SGN_OK;
}

static int factor_numeric_impl(sgn_factor f, const double* d_values, int64_t values_stride,
                               double eps_x, double eps_lambda, const double* d_eps_x,
                               const double* d_eps_l, void* stream);

int sgn_factor_numeric(sgn_factor f, const double* d_values, int64_t values_stride, double eps_x,
                       double eps_lambda, void* stream) {
  return factor_numeric_impl(f, d_values, values_stride, eps_x, eps_lambda, nullptr, nullptr, stream);
}

int sgn_factor_numeric_v(sgn_factor f, const double* d_values, int64_t values_stride,
                         const double* d_eps_x, const double* d_eps_lambda, void* stream) {
  return factor_numeric_impl(f, d_values, values_stride, 0.0, 0.0, d_eps_x, d_eps_lambda, stream);
}

static int factor_numeric_impl(sgn_factor f, const double* d_values, int64_t values_stride,
                               double eps_x, double eps_lambda, const double* d_eps_x,
                               const double* d_eps_l, void* stream) {
  const sgn::Symbolic& s = f->sym->s;
  cudaStream_t st = (cudaStream_t)stream;
  {
    std::vector<long long> init(f->batch, (long long)INT64_MAX);
    CUDA_TRY(cudaMemcpyAsync(f->status.p, init.data(), init.size() * sizeof(long long),
                             cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));  // keep `init` alive until the copy is done
  }
  for (const sgn::Launch& L : s.launches) {
    const dim3 grid((unsigned)L.count, f->batch);
    const Work* w = f->work.p + L.off;
    switch (L.kind) {
      case sgn::L_ASM:
        sgn::count_launch();
        k_assemble<<<grid, kAsmThreads, 0, st>>>(w, f->fronts.p, f->children.p, f->rel.p,
                                                 f->tile_ptr.p, f->tile_nnz.p, f->tile_loc.p,
                                                 f->kind_pos.p, d_values, values_stride, eps_x,
                                                 eps_lambda, d_eps_x, d_eps_l, f->fstore.p,
                                                 s.front_doubles);
        break;
      case sgn::L_PANEL:
        sgn::count_launch();
        if (L.pivtype == 2)
          k_panel<2><<<grid, kPanelThreads, 0, st>>>(w, f->fronts.p, f->perm.p, f->fstore.p,
                                                s.front_doubles, f->wstore.p, s.w_doubles,
                                                f->dscr.p, s.d_doubles, f->status.p);
        else
        k_panel<1><<<grid, kPanelThreads, 0, st>>>(w, f->fronts.p, f->perm.p, f->fstore.p,
                                                s.front_doubles, f->wstore.p, s.w_doubles,
                                                f->dscr.p, s.d_doubles, f->status.p);
        break;
      case sgn::L_ZPANEL:
        sgn::count_launch();
        k_zpanel<<<grid, kZThreads, 0, st>>>(w, f->fronts.p, f->fstore.p, s.front_doubles,
                                               f->zstore.p, s.z_doubles, f->dscr.p, s.d_doubles);
        break;
      case sgn::L_UPDATE:
        sgn::count_launch();
        k_update<<<grid, kUpdThreads, 0, st>>>(w, f->fronts.p, f->fstore.p, s.front_doubles,
                                               f->wstore.p, s.w_doubles);
        break;
    }
  }
  CUDA_TRY(cudaGetLastError());
  return SGN_OK;
}

int sgn_factor_check(sgn_factor f, void* stream, int64_t* pivot_index) {
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<long long> h(f->batch);
  CUDA_TRY(cudaMemcpyAsync(h.data(), f->status.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (long long v : h)
    if (v != (long long)INT64_MAX) {
      if (pivot_index) *pivot_index = v;
      sgn::last_error() = "zero pivot at unknown " + std::to_string(v);
      return SGN_SINGULAR;
    }
  if (pivot_index) *pivot_index = -1;
  return SGN_OK;
}

int sgn_factor_status(sgn_factor f, void* stream, int64_t* pivots) {
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<long long> h(f->batch);
  CUDA_TRY(cudaMemcpyAsync(h.data(), f->status.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int b = 0; b < f->batch; ++b) pivots[b] = (h[b] == (long long)INT64_MAX) ? -1 : (int64_t)h[b];
  return SGN_OK;
}

int sgn_debug_solve_trace(sgn_factor f, int64_t* out, int64_t cap, int64_t* n_tasks, int32_t* meta) {
  const sgn::Symbolic& s = f->sym->s;
  const int64_t nt = (int64_t)s.stasks.size() * f->batch;
  if (n_tasks) *n_tasks = nt;
  if (meta) {   // per task: kind, front, level, a, b
    for (size_t t = 0; t < s.stasks.size(); ++t) {
      const sgn::Task& T = s.stasks[t];
      meta[5 * t] = T.kind; meta[5 * t + 1] = T.f; meta[5 * t + 2] = s.fronts[T.f].level;
      meta[5 * t + 3] = T.a; meta[5 * t + 4] = T.b;
    }
  }
  if (out && f->trace.p) {
    const int64_t m = std::min<int64_t>(cap, 6 * nt);
    CUDA_TRY(cudaMemcpy(out, f->trace.p, m * sizeof(int64_t), cudaMemcpyDeviceToHost));
  }
  return SGN_OK;
}

int sgn_factor_solve(sgn_factor f, const double* d_b, double* d_x, int32_t flags, void* stream) {
  return launch_solve(f, d_b, d_x, flags, (cudaStream_t)stream);
}

void sgn_factor_destroy(sgn_factor f) { delete f; }

int sgn_spmv(sgn_factor f, const double* d_values, int64_t values_stride, const double* d_x,
             double* d_y, int32_t flags, void* stream) {
  return launch_spmv(f, d_values, values_stride, d_x, d_y, flags, (cudaStream_t)stream);
}

int sgn_solve_refined(sgn_factor f, const double* d_values, int64_t values_stride,
                      const double* d_rhs, double* d_sol, double tol, int32_t max_iters,
                      int32_t flags, double* rel_res, int32_t* iters, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = f->n;
  const int B = f->batch;
  const size_t N = (size_t)B * std::max<int64_t>(n, 1);
  int rc;
  if (!f->bicg_ready) {
    if ((rc = f->bx.alloc(N)) || (rc = f->br.alloc(N)) || (rc = f->brh.alloc(N)) ||
        (rc = f->bp.alloc(N)) || (rc = f->bv.alloc(N)) || (rc = f->bs.alloc(N)) ||
        (rc = f->bt.alloc(N)) || (rc = f->btmp.alloc(N)) || (rc = f->bbest.alloc(N)) ||
        (rc = f->bb.alloc(N)) || (rc = f->bscr.alloc(N)) ||
        (rc = f->partial.alloc((size_t)B * kDotBlocks * 2)) || (rc = f->bst.alloc(B)))
      return rc;
    f->bicg_ready = true;
  }
  const dim3 vg((unsigned)std::min<int64_t>((n + 255) / 256, 1024), B);
  const dim3 dg(kDotBlocks, B);
  BiState* S = f->bst.p;
  auto dot = [&](const double* a, const double* b2, const double* c, const double* d, int step, int it) {
    sgn::count_launch();
    k_dot_partial<<<dg, kDotThreads, 0, st>>>(a, b2, c, d, n, f->partial.p);
    sgn::count_launch();
    k_dot_final<<<B, 32, 0, st>>>(f->partial.p, S, step, tol, it);
  };
  // vectors: bb = b, bx = x, br = r, brh = r_hat, bp = p, bv = v, bs = s, bt = t,
  //          btmp = b - A x, bscr = A * (.), bbest = best iterate
  CUDA_TRY(cudaMemcpyAsync(f->bb.p, d_rhs, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const sgn::Symbolic& sy = f->sym->s;
  if ((flags & SGN_SOLVE_LEADING) && sy.pair_mode && sy.n_p > 0) {
    for (int b = 0; b < B; ++b)
      CUDA_TRY(cudaMemsetAsync(f->bb.p + (size_t)b * n + sy.n_x, 0, sy.n_p * sizeof(double), st));
  }
  dot(f->bb.p, f->bb.p, nullptr, nullptr, 0, 0);                                   // bnorm
  if ((rc = launch_solve(f, f->bb.p, f->bx.p, flags, st))) return rc;              // x0
  if ((rc = launch_spmv(f, d_values, values_stride, f->bx.p, f->bscr.p, flags, st))) return rc;
  sgn::count_launch();
  k_vec<<<vg, 256, 0, st>>>(0, S, n, f->btmp.p, f->bb.p, f->bscr.p, nullptr, nullptr, nullptr);
  dot(f->btmp.p, f->btmp.p, nullptr, nullptr, 1, 0);                               // res0
  sgn::count_launch();
  k_vec<<<vg, 256, 0, st>>>(9, S, n, f->bbest.p, f->bx.p, nullptr, nullptr, nullptr, nullptr);
  std::vector<BiState> hs(B);
  auto read_state = [&]() -> int {
    CUDA_TRY(cudaMemcpyAsync(hs.data(), S, B * sizeof(BiState), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return 0;
  };
  if ((rc = read_state())) return rc;
  bool any = false;
  for (auto& h : hs) any |= (h.active != 0);
  if (any && max_iters > 0) {
    if ((rc = launch_solve(f, f->btmp.p, f->br.p, flags, st))) return rc;          // r = M^-1(b-Ax0)
    sgn::count_launch();
    k_vec<<<vg, 256, 0, st>>>(4, S, n, f->brh.p, f->br.p, nullptr, nullptr, nullptr, nullptr);
    CUDA_TRY(cudaMemsetAsync(f->bp.p, 0, N * sizeof(double), st));
    CUDA_TRY(cudaMemsetAsync(f->bv.p, 0, N * sizeof(double), st));
    for (int it = 1; it <= max_iters; ++it) {
      dot(f->brh.p, f->br.p, nullptr, nullptr, 2, it);                             // rho, beta
      sgn::count_launch();
      k_vec<<<vg, 256, 0, st>>>(1, S, n, f->bp.p, f->br.p, f->bv.p, nullptr, nullptr, nullptr);
      if ((rc = launch_spmv(f, d_values, values_stride, f->bp.p, f->bscr.p, flags, st))) return rc;
      if ((rc = launch_solve(f, f->bscr.p, f->bv.p, flags, st))) return rc;        // v = M^-1 A p
      dot(f->brh.p, f->bv.p, nullptr, nullptr, 3, it);                             // alpha
      sgn::count_launch();
      k_vec<<<vg, 256, 0, st>>>(2, S, n, f->bs.p, f->br.p, f->bv.p, nullptr, nullptr, nullptr);
      if ((rc = launch_spmv(f, d_values, values_stride, f->bs.p, f->bscr.p, flags, st))) return rc;
      if ((rc = launch_solve(f, f->bscr.p, f->bt.p, flags, st))) return rc;        // t = M^-1 A s
      dot(f->bt.p, f->bt.p, f->bt.p, f->bs.p, 4, it);                              // omega
      sgn::count_launch();
      k_vec<<<vg, 256, 0, st>>>(3, S, n, f->bx.p, f->bp.p, f->bs.p, f->bt.p, f->br.p, nullptr);
      if ((rc = launch_spmv(f, d_values, values_stride, f->bx.p, f->bscr.p, flags, st))) return rc;
      sgn::count_launch();
      k_vec<<<vg, 256, 0, st>>>(0, S, n, f->btmp.p, f->bb.p, f->bscr.p, nullptr, nullptr, nullptr);
      dot(f->btmp.p, f->btmp.p, nullptr, nullptr, 5, it);                          // true residual
      sgn::count_launch();
      k_vec<<<vg, 256, 0, st>>>(7, S, n, f->bbest.p, f->bx.p, nullptr, nullptr, nullptr, nullptr);
      sgn::count_launch();
      k_clear_reason<<<B, 32, 0, st>>>(S);
      if ((rc = read_state())) return rc;
      bool act = false;
      for (auto& h : hs) act |= (h.active != 0);
      if (!act) break;
    }
  }
  sgn::count_launch();
  k_select<<<vg, 256, 0, st>>>(S, n, f->bx.p, f->bbest.p, d_sol);
  CUDA_TRY(cudaGetLastError());
  if ((rc = read_state())) return rc;
  bool fail = false;
  for (int b = 0; b < B; ++b) {
    const BiState& h = hs[b];
    const double res = (h.reason == 1 || h.reason == 4) ? h.res : h.best_res;
    const int32_t its = h.active ? max_iters : h.iters;
    if (rel_res) rel_res[b] = res;
    if (iters) iters[b] = its;
    if (!(res <= tol)) fail = true;
  }
  if (fail) {
    sgn::last_error() = "BiCGSTAB refinement stalled above tolerance";
    return SGN_NO_CONVERGENCE;
  }
  return SGN_OK;
}

}  // extern "C"
