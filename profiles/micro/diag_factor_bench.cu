// Microbenchmark: cycles for one 32x32 LDL^T diagonal-block factorization by one warp
// (variants of factor_diag in paper_2107_03285_b200/csrc/factor_dag.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o diag_bench diag_factor_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kTile = 32;

template <int PT, bool RCP>
__device__ int fd_window(double (*D)[kTile + 1], double2* colbuf, int w) {
  const int i = threadIdx.x & 31;
  double d[kTile];
#pragma unroll
  for (int m = 0; m < kTile; ++m) d[m] = (m <= i) ? D[i][m] : 0.0;
  int first_bad = 1 << 30;
  for (int j = 0; j < w; j += PT) {
    colbuf[i] = make_double2(d[0], PT == 2 ? d[1] : 0.0);
    __syncwarp();
    double l0 = 0.0, l1 = 0.0;
    const bool below = (i >= j + PT) && (i < w);
    if (PT == 2) {
      const double2 pj = colbuf[j], pj1 = colbuf[j + 1];
      const double a = pj.x, bb = pj1.x, c = pj1.y;
      double det = a * c - bb * bb;
      const bool badp = (det == 0.0 || !isfinite(det));
      if (badp && first_bad > j) first_bad = j;
      if (badp) det = 1.0;
      const double rdet = RCP ? __drcp_rn(det) : 1.0 / det;
      const double ia = c * rdet, ib = -bb * rdet, ic = a * rdet;
      if (below) { l0 = d[0] * ia + d[1] * ib; l1 = d[0] * ib + d[1] * ic; }
#pragma unroll
      for (int m = 2; m < kTile; ++m)
        if (j + m < kTile) {
          const double2 y = colbuf[j + m];
          d[m] -= l0 * y.x + l1 * y.y;
        }
      if (below) { D[i][j] = l0; D[i][j + 1] = l1; }
      else if (i == j) D[j][j] = d[0];
      else if (i == j + 1) { D[j + 1][j] = d[0]; D[j + 1][j + 1] = d[1]; }
    } else {
      double dj = colbuf[j].x;
      const bool badp = (dj == 0.0 || !isfinite(dj));
      if (badp && first_bad > j) first_bad = j;
      if (badp) dj = 1.0;
      const double rd = RCP ? __drcp_rn(dj) : 1.0 / dj;
      if (below) l0 = d[0] * rd;
#pragma unroll
      for (int m = 1; m < kTile; ++m)
        if (j + m < kTile) d[m] -= l0 * colbuf[j + m].x;
      if (below) D[i][j] = l0;
      else if (i == j) D[j][j] = d[0];
    }
#pragma unroll
    for (int m = 0; m + PT < kTile; ++m) d[m] = d[m + PT];
    __syncwarp();
  }
  return first_bad;
}

template <int PT>
__device__ int fd_smem(double (*D)[kTile + 1], int w) {
  const int i = threadIdx.x & 31;
  int first_bad = 1 << 30;
  for (int j = 0; j < w; j += PT) {
    if (PT == 2) {
      const double a = D[j][j], bb = D[j + 1][j], c = D[j + 1][j + 1];
      double det = a * c - bb * bb;
      if ((det == 0.0 || !isfinite(det)) && first_bad > j) first_bad = j;
      const double rdet = 1.0 / det;
      const double ia = c * rdet, ib = -bb * rdet, ic = a * rdet;
      const bool below = (i > j + 1) && (i < w);
      const double x0 = below ? D[i][j] : 0.0, x1 = below ? D[i][j + 1] : 0.0;
      const double l0 = x0 * ia + x1 * ib, l1 = x0 * ib + x1 * ic;
#pragma unroll 4
      for (int k = j + 2; k < w; ++k) {
        const double y0 = D[k][j], y1 = D[k][j + 1];
        if (below && k <= i) D[i][k] -= l0 * y0 + l1 * y1;
      }
      __syncwarp();
      if (below) { D[i][j] = l0; D[i][j + 1] = l1; }
      __syncwarp();
    } else {
      const double dj = D[j][j];
      const double rd = 1.0 / dj;
      const bool below = (i > j) && (i < w);
      const double l = below ? D[i][j] * rd : 0.0;
#pragma unroll 4
      for (int k = j + 1; k < w; ++k) {
        const double y = D[k][j];
        if (below && k <= i) D[i][k] -= l * y;
      }
      __syncwarp();
      if (below) D[i][j] = l;
      __syncwarp();
    }
  }
  return first_bad;
}

// fully unrolled, rows in registers, shuffles (the round-1 level-kernel scheme)
template <int PT>
__device__ int fd_unrolled(double (*D)[kTile + 1], int w) {
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
        d[k] -= l0 * y0 + l1 * y1;
      }
      d[j] = below ? l0 : d[j];
      d[j + 1] = below ? l1 : d[j + 1];
    } else {
      double dj = __shfl_sync(0xffffffffu, d[j], j);
      dj = act ? dj : 1.0;
      const bool below = act && (i > j) && (i < w);
      const double x = d[j];
      const double l = below ? x * (1.0 / dj) : 0.0;
#pragma unroll
      for (int k = j + 1; k < kTile; ++k) {
        const double y = __shfl_sync(0xffffffffu, x, k);
        d[k] -= l * y;
      }
      d[j] = below ? l : d[j];
    }
  }
#pragma unroll
  for (int k = 0; k < kTile; ++k) if (k <= i) D[i][k] = d[k];
  return first_bad;
}


// window variant with a 64-entry zero-padded broadcast buffer (no per-element guards)
template <int PT>
__device__ int fd_window_pad(double (*D)[kTile + 1], double2* colbuf, int w) {
  const int i = threadIdx.x & 31;
  double d[kTile];
#pragma unroll
  for (int m = 0; m < kTile; ++m) d[m] = (m <= i) ? D[i][m] : 0.0;
  colbuf[kTile + i] = make_double2(0.0, 0.0);
  int first_bad = 1 << 30;
  for (int j = 0; j < w; j += PT) {
    colbuf[i] = make_double2(d[0], PT == 2 ? d[1] : 0.0);
    __syncwarp();
    double l0 = 0.0, l1 = 0.0;
    const bool below = (i >= j + PT) && (i < w);
    const double2* cb = colbuf + j;
    if (PT == 2) {
      const double2 pj = cb[0], pj1 = cb[1];
      const double a = pj.x, bb = pj1.x, c = pj1.y;
      double det = a * c - bb * bb;
      const bool badp = (det == 0.0 || !isfinite(det));
      if (badp && first_bad > j) first_bad = j;
      if (badp) det = 1.0;
      const double rdet = 1.0 / det;
      const double ia = c * rdet, ib = -bb * rdet, ic = a * rdet;
      if (below) { l0 = d[0] * ia + d[1] * ib; l1 = d[0] * ib + d[1] * ic; }
#pragma unroll
      for (int m = 2; m < kTile; ++m) {
        const double2 y = cb[m];
        d[m] = fma(-l1, y.y, fma(-l0, y.x, d[m]));
      }
      if (below) { D[i][j] = l0; D[i][j + 1] = l1; }
      else if (i == j) D[j][j] = d[0];
      else if (i == j + 1) { D[j + 1][j] = d[0]; D[j + 1][j + 1] = d[1]; }
    } else {
      double dj = cb[0].x;
      const bool badp = (dj == 0.0 || !isfinite(dj));
      if (badp && first_bad > j) first_bad = j;
      if (badp) dj = 1.0;
      const double rd = 1.0 / dj;
      if (below) l0 = d[0] * rd;
#pragma unroll
      for (int m = 1; m < kTile; ++m) d[m] = fma(-l0, cb[m].x, d[m]);
      if (below) D[i][j] = l0;
      else if (i == j) D[j][j] = d[0];
    }
#pragma unroll
    for (int m = 0; m + PT < kTile; ++m) d[m] = d[m + PT];
    __syncwarp();
  }
  return first_bad;
}

// fully unrolled, rows in registers, pivot columns broadcast through smem (no shuffles)
template <int PT>
__device__ int fd_unrolled_smem(double (*D)[kTile + 1], double2* colbuf, int w) {
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
      det = act ? det : 1.0;
      const double rdet = 1.0 / det;
      const double ia = c * rdet, ib = -bb * rdet, ic = a * rdet;
      const bool below = act && (i > j + 1) && (i < w);
      const double x0 = d[j], x1 = d[j + 1];
      const double l0 = below ? x0 * ia + x1 * ib : 0.0;
      const double l1 = below ? x0 * ib + x1 * ic : 0.0;
#pragma unroll
      for (int k = j + 2; k < kTile; ++k) {
        const double2 y = colbuf[k];
        d[k] = fma(-l1, y.y, fma(-l0, y.x, d[k]));
      }
      d[j] = below ? l0 : d[j];
      d[j + 1] = below ? l1 : d[j + 1];
    } else {
      double dj = colbuf[j].x;
      dj = act ? dj : 1.0;
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

template <int V, int PT>
__global__ void kbench(const double* in, double* out, long long* cyc, int reps, int wr) {
  __shared__ double D[kTile][kTile + 1];
  __shared__ double2 colbuf[2 * kTile];
  const int i = threadIdx.x;
  long long total = 0;
  int bad = 0;
  for (int r = 0; r < reps; ++r) {
    for (int k = 0; k < kTile; ++k) D[i][k] = in[i * kTile + k];
    __syncwarp();
    const long long t0 = clock64();
    if (V == 0) bad += fd_window<PT, false>(D, colbuf, kTile);
    else if (V == 1) bad += fd_window<PT, true>(D, colbuf, kTile);
    else if (V == 2) bad += fd_smem<PT>(D, kTile);
    else if (V == 3) bad += fd_unrolled<PT>(D, kTile);
    else if (V == 4) bad += fd_window_pad<PT>(D, colbuf, wr);
    else bad += fd_unrolled_smem<PT>(D, colbuf, wr);
    __syncwarp();
    const long long t1 = clock64();
    total += t1 - t0;
  }
  for (int k = 0; k < kTile; ++k) out[i * kTile + k] = D[i][k];
  if (i == 0) { cyc[0] = total / reps; cyc[1] = bad; }
}

int main(int argc, char** argv) {
  const int wr = argc > 1 ? atoi(argv[1]) : 32;
  double h[kTile * kTile];
  for (int i = 0; i < kTile; ++i)
    for (int k = 0; k < kTile; ++k) {
      double v = 1.0 / (1.0 + i + k) + ((i == k) ? ((i & 1) ? -4.0 : 4.0) : 0.0);
      h[i * kTile + k] = v;
    }
  double *din, *dout;
  long long* dc;
  cudaMalloc(&din, sizeof h); cudaMalloc(&dout, sizeof h); cudaMalloc(&dc, 16);
  cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
  const char* names[] = {"window/div", "window/rcp", "smem-loop", "unrolled-shfl", "window-pad", "unrolled-smem"};
  double ref[kTile * kTile];
  for (int pt = 1; pt <= 2; ++pt)
    for (int v = 0; v < 6; ++v) {
      long long c[2];
      double o[kTile * kTile];
      for (int rep = 0; rep < 2; ++rep) {
        if (pt == 1) {
          if (v == 0) kbench<0, 1><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 1) kbench<1, 1><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 2) kbench<2, 1><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 3) kbench<3, 1><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 4) kbench<4, 1><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 5) kbench<5, 1><<<1, 32>>>(din, dout, dc, 20, wr);
        } else {
          if (v == 0) kbench<0, 2><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 1) kbench<1, 2><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 2) kbench<2, 2><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 3) kbench<3, 2><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 4) kbench<4, 2><<<1, 32>>>(din, dout, dc, 20, wr);
          if (v == 5) kbench<5, 2><<<1, 32>>>(din, dout, dc, 20, wr);
        }
        cudaDeviceSynchronize();
      }
      cudaMemcpy(c, dc, 16, cudaMemcpyDeviceToHost);
      cudaMemcpy(o, dout, sizeof o, cudaMemcpyDeviceToHost);
      if (v == 0) for (int q = 0; q < kTile * kTile; ++q) ref[q] = o[q];
      double md = 0;
      for (int i = 0; i < kTile; ++i)
        for (int k = 0; k <= i; ++k) {
          double dd = o[i * kTile + k] - ref[i * kTile + k];
          if (dd < 0) dd = -dd;
          if (dd > md) md = dd;
        }
      printf("PT=%d %-14s cycles %6lld  maxdiff vs window/div %.3e  bad %lld\n", pt, names[v], c[0], md, c[1]);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
