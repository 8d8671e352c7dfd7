// Microbenchmark: Schur-update tile bodies of the persistent factorization on the FP64
// tensor pipe (mma.sync.m8n8k4.f64 -> DMMA), all SMs, 4 CTAs x 128 threads per SM (the
// persistent kernel's shape).  Each task: C(tile) -= sum over ns pivot steps of
// L21(rows, step) W(cols, step)^T, operands read from an L2-resident column-major "front".
//   v32   : 32x32 C tile, warps 8x32, register prefetch of the next step (factor_dag.cu f_update)
//   v64   : 64x64 C tile, warps 32x32 (4x4 fragments), C in registers, staged 32-wide steps
//   v64a  : 64x64 C tile, cp.async.cg 16-byte double buffer of 16-wide half steps (aligned ld)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o upd_bench upd_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

constexpr int LD = 2048;          // front leading dimension (rows)
constexpr int NS = 8;             // pivot steps per task

__device__ __forceinline__ void task_coords(int t, int tile, int& lo_i, int& lo_j, int& j0) {
  const int nb = (LD - 512) / tile;
  const int a = t % nb, b = (t / nb) % nb;
  lo_i = 512 + a * tile;
  lo_j = 512 + b * tile;
  j0 = 32 * ((t / (nb * nb)) % 4);
}

// ---------------------------------------------------------------------------- v32
__global__ void __launch_bounds__(128, 4) k_v32(double* F, int ntask) {
  __shared__ double Ak[32][40], Bk[32][40], Cs[32][40];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int row0 = warp * 8, i = row0 + g;
  for (int t = blockIdx.x; t < ntask; t += gridDim.x) {
    int lo_i, lo_j, j0;
    task_coords(t, 32, lo_i, lo_j, j0);
    double va[8], vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = tid + u * 128, r = e & 31, c = e >> 5;
      Cs[c][r] = __ldcg(F + (size_t)(lo_j + c) * LD + lo_i + r);
    }
#define LOADS(S_)                                                                  \
    _Pragma("unroll") for (int u = 0; u < 8; ++u) {                                \
      const int e = tid + u * 128, r = e & 31, c = e >> 5;                         \
      va[u] = __ldcg(F + (size_t)(j0 + 32 * (S_) + c) * LD + lo_i + r);            \
      vb[u] = __ldcg(F + (size_t)(lo_j + c) * LD + j0 + 32 * (S_) + r);            \
    }
    LOADS(0);
    double acc[4][2] = {};
    for (int s = 0; s < NS; ++s) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = tid + u * 128, r = e & 31, c = e >> 5;
        Ak[c][r] = va[u];
        Bk[r][c] = vb[u];
      }
      __syncthreads();
      if (s + 1 < NS) { LOADS(s + 1); }
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        const double a = Ak[kk + q][row0 + g];
#pragma unroll
        for (int nf = 0; nf < 4; ++nf) dmma(acc[nf][0], acc[nf][1], a, Bk[kk + q][nf * 8 + g]);
      }
      __syncthreads();
    }
#undef LOADS
#pragma unroll
    for (int nf = 0; nf < 4; ++nf)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = nf * 8 + 2 * q + h;
        F[(size_t)(lo_j + j) * LD + lo_i + i] = Cs[j][i] - acc[nf][h];
      }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------- v64
__global__ void __launch_bounds__(128, 4) k_v64(double* F, int ntask) {
  __shared__ double As[32][68], Bs[64][36];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  for (int t = blockIdx.x; t < ntask; t += gridDim.x) {
    int lo_i, lo_j, j0;
    task_coords(t, 64, lo_i, lo_j, j0);
    double acc[4][4][2];
#pragma unroll
    for (int mf = 0; mf < 4; ++mf)
#pragma unroll
      for (int nf = 0; nf < 4; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          acc[mf][nf][h] = 0.0;
    for (int s = 0; s < NS; ++s) {
      const int k0 = j0 + 32 * s;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = tid + (u + 8 * hh) * 128, r = e & 63, c = e >> 6;
          v[u] = __ldcg(F + (size_t)(k0 + c) * LD + lo_i + r);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = tid + (u + 8 * hh) * 128, r = e & 63, c = e >> 6;
          As[c][r] = v[u];
        }
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = tid + (u + 8 * hh) * 128, r = e & 31, c = e >> 5;
          v[u] = __ldcg(F + (size_t)(lo_j + c) * LD + k0 + r);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = tid + (u + 8 * hh) * 128, r = e & 31, c = e >> 5;
          Bs[c][r] = v[u];
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 32; kk += 4) {
        double a[4], b[4];
#pragma unroll
        for (int mf = 0; mf < 4; ++mf) a[mf] = As[kk + q][wm + 8 * mf + g];
#pragma unroll
        for (int nf = 0; nf < 4; ++nf) b[nf] = Bs[wn + 8 * nf + g][kk + q];
#pragma unroll
        for (int mf = 0; mf < 4; ++mf)
#pragma unroll
          for (int nf = 0; nf < 4; ++nf) dmma(acc[mf][nf][0], acc[mf][nf][1], a[mf], b[nf]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int mf = 0; mf < 4; ++mf)
#pragma unroll
      for (int nf = 0; nf < 4; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h)
        {
          double* p = F + (size_t)(lo_j + wn + 8 * nf + 2 * q + h) * LD + lo_i + wm + 8 * mf + g;
          *p = __ldcg(p) - acc[mf][nf][h];
        }
  }
}

// ---------------------------------------------------------------------------- v64a
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(128, 4) k_v64a(double* F, int ntask) {
  __shared__ __align__(16) double As[2][16][68];
  __shared__ __align__(16) double Bs[2][64][20];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, q = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  for (int t = blockIdx.x; t < ntask; t += gridDim.x) {
    int lo_i, lo_j, j0;
    task_coords(t, 64, lo_i, lo_j, j0);
    auto issue = [&](int hs, int buf) {            // half step hs: k columns j0 + 16 hs ..
      const int k0 = j0 + 16 * hs;
#pragma unroll
      for (int u = 0; u < 4; ++u) {                // A: 16 cols x 64 rows = 512 chunks
        const int e = tid + u * 128, ch = e & 31, c = e >> 5;
        cp16(&As[buf][c][2 * ch], F + (size_t)(k0 + c) * LD + lo_i + 2 * ch);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {                // B: 64 rows x 16 k = 512 chunks
        const int e = tid + u * 128, ch = e & 7, j = e >> 3;
        cp16(&Bs[buf][j][2 * ch], F + (size_t)(lo_j + j) * LD + k0 + 2 * ch);
      }
      cp_commit();
    };
    issue(0, 0);
    double acc[4][4][2];
#pragma unroll
    for (int mf = 0; mf < 4; ++mf)
#pragma unroll
      for (int nf = 0; nf < 4; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[mf][nf][h] = 0.0;
    for (int hs = 0; hs < 2 * NS; ++hs) {
      const int buf = hs & 1;
      if (hs + 1 < 2 * NS) { issue(hs + 1, buf ^ 1); cp_wait<1>(); } else { cp_wait<0>(); }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 16; kk += 4) {
        double a[4], b[4];
#pragma unroll
        for (int mf = 0; mf < 4; ++mf) a[mf] = As[buf][kk + q][wm + 8 * mf + g];
#pragma unroll
        for (int nf = 0; nf < 4; ++nf) b[nf] = Bs[buf][wn + 8 * nf + g][kk + q];
#pragma unroll
        for (int mf = 0; mf < 4; ++mf)
#pragma unroll
          for (int nf = 0; nf < 4; ++nf) dmma(acc[mf][nf][0], acc[mf][nf][1], a[mf], b[nf]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int mf = 0; mf < 4; ++mf)
#pragma unroll
      for (int nf = 0; nf < 4; ++nf)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double* p = F + (size_t)(lo_j + wn + 8 * nf + 2 * q + h) * LD + lo_i + wm + 8 * mf + g;
          *p = __ldcg(p) - acc[mf][nf][h];
        }
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* F;
  cudaMalloc(&F, (size_t)LD * LD * sizeof(double));
  cudaMemset(F, 0, (size_t)LD * LD * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"v32 (32x32, register prefetch)", "v64 (64x64, staged)", "v64a (64x64, cp.async x2)"};
  for (int v = 0; v < 3; ++v) {
    for (int ctas_per_sm : {4, 2}) {
      const int tile = v == 0 ? 32 : 64;
      const int ntask = (v == 0 ? 64 : 16) * sms * 4 * 4;
      const int grid = sms * ctas_per_sm;
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (v == 0) k_v32<<<grid, 128>>>(F, ntask);
        else if (v == 1) k_v64<<<grid, 128>>>(F, ntask);
        else k_v64a<<<grid, 128>>>(F, ntask);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      const double flops = (double)ntask * NS * 2.0 * tile * tile * 32;
      printf("%-34s %d CTA/SM: %8.3f ms  %6.2f TFLOP/s  (%s)\n", names[v], ctas_per_sm, best,
             flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
