// Dense Gauss-Newton (DGN) building blocks on B200: the caller-side
// alternative direction of the reference, reference optimize.py:168-198:
//   S = -G_x^{-1} G_p          sensitivity.py:167-178   (multi-RHS solve, numeric.cu)
//   H = S^T A S + B S + (B S)^T + C, symmetrised        sensitivity.py:232-242  (here)
//   dp = -H^{-1} g by a dense factorization             linear_solvers.py:214-240 (the
//        multifrontal LDL^T of numeric.cu on a dense pattern, positive pivots checked)
// Blocks of the stacked KKT K = [[A, B^T, G_x^T], [B, C, G_p^T], [G_x, G_p, 0]] are read
// straight from its device CSC (symmetric, so CSC == CSR).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <string>
#include <vector>

#include "../../include/sgn_b200.h"
#include "sgn_internal.h"

namespace {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// out (column-major, nr x nc, ld = nr) = K[r0:r0+nr, c0:c0+nc]; out pre-zeroed
__global__ void k_csc_block_dense(const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                                  const double* __restrict__ val, int64_t r0, int64_t nr, int64_t c0,
                                  int64_t nc, double* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nc; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = c0 + j;
    for (int64_t t = ptr[c]; t < ptr[c + 1]; ++t) {
      const int64_t r = idx[t] - r0;
      if (r >= 0 && r < nr) out[j * nr + r] = val[t];
    }
  }
}

// Y[j][r] = sum_c K[r0 + r, c0 + c] X[j][c] for r < nr, j < m (X[j], Y[j] contiguous of
// length ldx / ldy).  One thread per (r, j); K row r0 + r is column r0 + r (symmetric).
__global__ void k_csc_spmm(const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                           const double* __restrict__ val, int64_t r0, int64_t nr, int64_t c0, int64_t ncol,
                           const double* __restrict__ X, int64_t ldx, double* __restrict__ Y, int64_t ldy,
                           int64_t m) {
  const int64_t total = nr * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % nr, j = e / nr;
    const int64_t row = r0 + r;
    double s = 0.0;
    for (int64_t t = ptr[row]; t < ptr[row + 1]; ++t) {
      const int64_t c = idx[t] - c0;
      if (c >= 0 && c < ncol) s += val[t] * X[j * ldx + c];
    }
    Y[j * ldy + r] = s;
  }
}

// C[i][j] (column-major n x n) = sum_k X[i][k] Y[j][k]   (X, Y: n rows of length K, row-major)
// One 32x32 output tile per CTA, K in 32-chunks staged K-major (stride 40) in smem; DMMA.
constexpr int kGemmThreads = 128;
__global__ void __launch_bounds__(kGemmThreads)
k_gemm_tn(const double* __restrict__ X, const double* __restrict__ Y, int64_t n, int64_t K,
          double* __restrict__ C) {
  __shared__ double Ak[32][40];
  __shared__ double Bk[32][40];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int64_t i0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 32;
  double acc[4][2];
#pragma unroll
  for (int nf = 0; nf < 4; ++nf) acc[nf][0] = acc[nf][1] = 0.0;
  for (int64_t k0 = 0; k0 < K; k0 += 32) {
    double va[8], vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * kGemmThreads, kk = e & 31, r = e >> 5;
      const bool kin = k0 + kk < K;
      va[u] = (kin && i0 + r < n) ? X[(i0 + r) * K + k0 + kk] : 0.0;
      vb[u] = (kin && j0 + r < n) ? Y[(j0 + r) * K + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * kGemmThreads, kk = e & 31, r = e >> 5;
      Ak[kk][r] = va[u];
      Bk[kk][r] = vb[u];
    }
    __syncthreads();
    const int row0 = warp * 8;
#pragma unroll
    for (int kk = 0; kk < 32; kk += 4) {
      const double a = Ak[kk + q][row0 + g];
#pragma unroll
      for (int nf = 0; nf < 4; ++nf) dmma_8x8x4(acc[nf][0], acc[nf][1], a, Bk[kk + q][nf * 8 + g]);
    }
  }
  const int64_t i = i0 + warp * 8 + g;
#pragma unroll
  for (int nf = 0; nf < 4; ++nf)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = j0 + nf * 8 + 2 * q + h;
      if (i < n && j < n) C[j * n + i] = acc[nf][h];
    }
}

// H = 0.5 (M + M^T), M = STAS + BS + BS^T + C   (all column-major n x n; BS[i + n j] = (B S)[i][j])
__global__ void k_gn_hessian(const double* __restrict__ stas, const double* __restrict__ bs,
                             const double* __restrict__ c, int64_t n, double* __restrict__ H) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    const double mij = stas[j * n + i] + bs[j * n + i] + bs[i * n + j] + c[j * n + i];
    const double mji = stas[i * n + j] + bs[i * n + j] + bs[j * n + i] + c[i * n + j];
    H[e] = 0.5 * (mij + mji);
  }
}

// per front: min over its 1x1 pivots D_rr (read from the published diagonal of the front)
__global__ void k_min_pivot(const sgn::DFront* __restrict__ fronts, const double* __restrict__ fstore,
                            double* __restrict__ out_min, int64_t* __restrict__ out_pos) {
  const sgn::DFront F = fronts[blockIdx.x];
  __shared__ double sm[256];
  __shared__ int64_t sp[256];
  double m = DBL_MAX;
  int64_t pos = -1;
  const double* Fm = fstore + F.foff;
  for (int r = threadIdx.x; r < F.npiv; r += blockDim.x) {
    const int64_t ld = sgn::front_ld(F.nrow);
    double d = Fm[(int64_t)r * ld + r];
    if (F.pivtype == 2) {       // 2x2 block [a b; b c]: the equivalent 1x1 pivots a, det / a
      const int re = r & ~1;
      const double a = Fm[(int64_t)re * ld + re], bb = Fm[(int64_t)re * ld + re + 1];
      const double c = Fm[(int64_t)(re + 1) * ld + re + 1];
      d = (r == re) ? a : (a != 0.0 ? (a * c - bb * bb) / a : DBL_MAX);   // a == 0: reported at re
    }
    if (d < m) { m = d; pos = F.first + r; }
  }
  sm[threadIdx.x] = m;
  sp[threadIdx.x] = pos;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s && sm[threadIdx.x + s] < sm[threadIdx.x]) {
      sm[threadIdx.x] = sm[threadIdx.x + s];
      sp[threadIdx.x] = sp[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out_min[blockIdx.x] = sm[0]; out_pos[blockIdx.x] = sp[0]; }
}

}  // namespace

#define DENSE_CHECK()                                                              \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      sgn::last_error() = std::string("dense kernel: ") + cudaGetErrorString(_e);  \
      return SGN_CUDA_ERROR;                                                       \
    }                                                                              \
  } while (0)

extern "C" {

int sgn_csc_block_dense(int64_t n_cols_total, const int64_t* d_ptr, const int64_t* d_idx, const double* d_val,
                        int64_t r0, int64_t nr, int64_t c0, int64_t nc, double* d_out, void* stream) {
  (void)n_cols_total;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(d_out, 0, (size_t)nr * nc * sizeof(double), st) != cudaSuccess) DENSE_CHECK();
  if (nc == 0) return SGN_OK;
  sgn::count_launch();
  k_csc_block_dense<<<(unsigned)std::min<int64_t>((nc + 127) / 128, 4096), 128, 0, st>>>(d_ptr, d_idx, d_val, r0, nr, c0, nc, d_out);
  DENSE_CHECK();
  return SGN_OK;
}

int sgn_csc_spmm(const int64_t* d_ptr, const int64_t* d_idx, const double* d_val, int64_t r0, int64_t nr,
                 int64_t c0, int64_t ncol, const double* d_X, int64_t ldx, double* d_Y, int64_t ldy, int64_t m,
                 void* stream) {
  const int64_t total = nr * m;
  if (total == 0) return SGN_OK;
  sgn::count_launch();
  k_csc_spmm<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256, 0, (cudaStream_t)stream>>>(
      d_ptr, d_idx, d_val, r0, nr, c0, ncol, d_X, ldx, d_Y, ldy, m);
  DENSE_CHECK();
  return SGN_OK;
}

int sgn_gemm_tn(const double* d_X, const double* d_Y, int64_t n, int64_t K, double* d_C, void* stream) {
  if (n == 0) return SGN_OK;
  const dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  sgn::count_launch();
  k_gemm_tn<<<grid, kGemmThreads, 0, (cudaStream_t)stream>>>(d_X, d_Y, n, K, d_C);
  DENSE_CHECK();
  return SGN_OK;
}

int sgn_gn_hessian(const double* d_stas, const double* d_bs, const double* d_c, int64_t n, double* d_H,
                   void* stream) {
  if (n == 0) return SGN_OK;
  sgn::count_launch();
  k_gn_hessian<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 65535), 256, 0, (cudaStream_t)stream>>>(
      d_stas, d_bs, d_c, n, d_H);
  DENSE_CHECK();
  return SGN_OK;
}

}  // extern "C"

namespace sgn {
int min_pivot(const DFront* d_fronts, int32_t n_fronts, const double* d_fstore, double* out_min, int64_t* out_pos,
              void* stream) {
  double* dm = nullptr;
  int64_t* dp = nullptr;
  if (cudaMalloc(&dm, n_fronts * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&dp, n_fronts * sizeof(int64_t)) != cudaSuccess) {
    if (dm) cudaFree(dm);
    last_error() = "cudaMalloc";
    return SGN_CUDA_ERROR;
  }
  count_launch();
  k_min_pivot<<<n_fronts, 256, 0, (cudaStream_t)stream>>>(d_fronts, d_fstore, dm, dp);
  std::vector<double> hm(n_fronts);
  std::vector<int64_t> hp(n_fronts);
  cudaError_t e = cudaMemcpyAsync(hm.data(), dm, n_fronts * sizeof(double), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hp.data(), dp, n_fronts * sizeof(int64_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  cudaFree(dm);
  cudaFree(dp);
  if (e != cudaSuccess) { last_error() = std::string("min pivot: ") + cudaGetErrorString(e); return SGN_CUDA_ERROR; }
  *out_min = DBL_MAX;
  *out_pos = -1;
  for (int32_t k = 0; k < n_fronts; ++k)
    if (hm[k] < *out_min) { *out_min = hm[k]; *out_pos = hp[k]; }
  return SGN_OK;
}
}  // namespace sgn
