// FP64 peak microbenchmarks for the factorization roofline (MEASURED_PEAKS.json carries
// only HBM and bf16 figures).  DMMA: register-resident mma.sync.m8n8k4.f64 chains across
// all SMs; DFMA: independent fma chains.  Timed with CUDA events on the given stream.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/sgn_b200.h"
#include "sgn_internal.h"

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_dmma_peak(int iters, double* out) {
  double acc[kChains][2];
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-9 * lane, b = 1.0 - 1e-9 * lane;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dfma_peak(int iters, double* out) {
  double acc[kChains];
  const double a = 1.0 + 1e-12 * threadIdx.x, b = 1e-13;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" {

// mode 0: DMMA (tensor pipe), 1: DFMA.  Returns achieved TFLOP/s in *tflops.
int sgn_fp64_peak(int32_t mode, int32_t iters, double* tflops, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) { sgn::last_error() = "cudaMalloc"; return SGN_CUDA_ERROR; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  for (int rep = 0; rep < 2; ++rep) {  // rep 0 = warm-up
    cudaEventRecord(e0, st);
    sgn::count_launch();
    if (mode == 0) k_dmma_peak<<<blocks, threads, 0, st>>>(iters, out);
    else k_dfma_peak<<<blocks, threads, 0, st>>>(iters, out);
    cudaEventRecord(e1, st);
  }
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32.0;
  const double flops = (mode == 0) ? warps * iters * kChains * 512.0
                                   : (double)blocks * threads * iters * kChains * 2.0;
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { sgn::last_error() = cudaGetErrorString(e); return SGN_CUDA_ERROR; }
  return SGN_OK;
}

}  // extern "C"
