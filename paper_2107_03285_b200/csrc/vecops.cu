// Small batched vector kernels of the SGN direction / forward-solve pipeline (sm_100a).
//
// Deterministic (fixed-order, one CTA per instance) reductions for energies,
// objectives, norms and dots; the least-squares objective terms of the problem
// contract (reference sensitivity.py:83-93); and the adjoint-gradient assembly
// g = df/dp + Gp^T lam, lam = -Gx^{-T} df/dx (reference sensitivity.py:181-198) from a
// leading-block KKT solve, producing the SGN right-hand side (0, -g, 0)
// (sensitivity.py:245-256).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <algorithm>
#include <mutex>
#include <string>

#include "../../include/sgn_b200.h"
#include "sgn_internal.h"

namespace {

constexpr int kRed = 512;

// max that propagates NaN like numpy's norm(., inf) (fmax would drop it)
__device__ __forceinline__ double nanmax(double a, double b) { return (a != a || b != b) ? (a + b) : fmax(a, b); }

template <int OP>  // 0 sum, 1 dot, 2 max-abs

__global__ void __launch_bounds__(kRed)
k_reduce(int64_t n, const double* __restrict__ a, const double* __restrict__ b, int64_t stride,
         double* __restrict__ out) {
  __shared__ double sh[kRed];
  const int inst = blockIdx.x;
  const double* ab = a + (int64_t)inst * stride;
  const double* bb = b ? b + (int64_t)inst * stride : nullptr;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kRed) {
    const double v = ab[i];
    if (OP == 0) acc += v;
    else if (OP == 1) acc += v * bb[i];
    else acc = nanmax(acc, fabs(v));
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kRed / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      if (OP == 2) sh[threadIdx.x] = nanmax(sh[threadIdx.x], sh[threadIdx.x + s]);
      else sh[threadIdx.x] += sh[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[inst] = sh[0];
}

__global__ void k_axpy(int64_t n, const double* __restrict__ alpha, const double* __restrict__ x,
                       const double* __restrict__ y, double* __restrict__ out, int64_t stride) {
  const int b = blockIdx.y;
  const double a = alpha[b];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = (int64_t)b * stride + i;
    out[k] = (y ? y[k] : 0.0) + a * x[k];
  }
}

// f vector (KKT order): x block = sigma w_t r at target dofs, p block = -R^T w_t r + w_reg p,
// lambda block 0, with r = sigma x[tdofs] - tvals - R p (R optional, CSR over targets; R^T is
// the CSR over parameters); objective per instance = 0.5 sum w r^2 + 0.5 w_reg |p|^2.
// Two grid-stride kernels (targets, then parameters: the R^T rows read the target
// residuals) on up to kLsqBlocks CTAs per instance; block partials are summed by the last
// CTA of the second kernel in block order (fixed tree: deterministic for any batch size).
constexpr int kLsqThreads = 256, kLsqBlocks = 64;
__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = kLsqThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

__global__ void __launch_bounds__(kLsqThreads)
k_lsq_targets(int64_t n_x, int64_t n_p, int64_t nt, const int64_t* __restrict__ tdofs,
              const double* __restrict__ tvals, int64_t tstride, double w_t, double xs, const double* __restrict__ x,
              const double* __restrict__ p, double* __restrict__ vec, const int64_t* __restrict__ rptr,
              const int64_t* __restrict__ ridx, const double* __restrict__ rcoef, double* __restrict__ rscr,
              double* __restrict__ part) {
  __shared__ double sh[kLsqThreads];
  const int b = blockIdx.y;
  const int64_t dim = 2 * n_x + n_p;
  double* v = vec ? vec + (int64_t)b * dim : nullptr;
  const double* xb = x + (int64_t)b * n_x;
  const double* pb = p + (int64_t)b * n_p;
  double* rs = rscr ? rscr + (int64_t)b * nt : nullptr;
  double acc = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)kLsqThreads + threadIdx.x; t < nt; t += (int64_t)gridDim.x * kLsqThreads) {
    const int64_t d = tdofs[t];
    double r = xs * xb[d] - tvals[(int64_t)b * tstride + t];
    if (rptr)
      for (int64_t k = rptr[t]; k < rptr[t + 1]; ++k) r -= rcoef[k] * pb[ridx[k]];
    acc += w_t * r * r;
    if (v) v[d] = xs * w_t * r;
    if (rs) rs[t] = w_t * r;
  }
  const double tot = block_sum(acc, sh);
  if (threadIdx.x == 0) part[((int64_t)b * 2 * kLsqBlocks) + blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kLsqThreads)
k_lsq_params(int64_t n_x, int64_t n_p, int64_t nt, int nbt, double w_reg, const double* __restrict__ p,
             double* __restrict__ vec, double* __restrict__ fobj, const int64_t* __restrict__ rtptr,
             const int64_t* __restrict__ rtidx, const double* __restrict__ rtcoef,
             const double* __restrict__ rscr, double* __restrict__ part, int* __restrict__ tickets) {
  __shared__ double sh[kLsqThreads];
  __shared__ int last;
  const int b = blockIdx.y;
  const int64_t dim = 2 * n_x + n_p;
  double* v = vec ? vec + (int64_t)b * dim : nullptr;
  const double* pb = p + (int64_t)b * n_p;
  const double* rs = rscr ? rscr + (int64_t)b * nt : nullptr;
  double acc = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)kLsqThreads + threadIdx.x; j < n_p; j += (int64_t)gridDim.x * kLsqThreads) {
    const double pj = pb[j];
    acc += w_reg * pj * pj;
    double fp = w_reg * pj;
    if (rtptr)
      for (int64_t k = rtptr[j]; k < rtptr[j + 1]; ++k) fp -= rtcoef[k] * rs[rtidx[k]];
    if (v) v[n_x + j] = fp;
  }
  const double tot = block_sum(acc, sh);
  double* pp = part + (int64_t)b * 2 * kLsqBlocks;
  if (threadIdx.x == 0) {
    pp[kLsqBlocks + blockIdx.x] = tot;
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(tickets + b) : "memory");
    last = (old == (int)gridDim.x - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  tickets[b] = 0;
  double t = 0.0;
  for (int k = 0; k < nbt; ++k) t += __ldcg(pp + k);
  for (int k = 0; k < (int)gridDim.x; ++k) t += __ldcg(pp + kLsqBlocks + k);
  if (fobj) fobj[b] = 0.5 * t;
}

// Rest-length residuals of 2-D springs (the reference spring bar's regularizer,
// spring_bar.py:159-184): r_s = |X_a - X_b| - L0_s, j_s = dr_s/dX = (d, -d), d the unit
// rest direction.  Per spring, out = [w j j^T (4 x 4, row-major) | w r j (4) | r^2], the
// element blocks the KKT gather sums into C = J_p^T W J_p and the f_p gather into w J_p^T r.
__global__ void k_restlen(int64_t ns, const int32_t* __restrict__ conn, const double* __restrict__ rest,
                          int64_t vstride, const double* __restrict__ L0, double w, double* __restrict__ out,
                          int64_t ostride) {
  const int b = blockIdx.y;
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const double* X = rest + (int64_t)b * vstride;
  const int va = conn[2 * s], vb = conn[2 * s + 1];
  const double dx = X[2 * va] - X[2 * vb], dy = X[2 * va + 1] - X[2 * vb + 1];
  const double len = sqrt(dx * dx + dy * dy);
  const double r = len - L0[s];
  const double j[4] = {dx / len, dy / len, -dx / len, -dy / len};
  double* o = out + (int64_t)b * ostride + s * 21;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
#pragma unroll
    for (int v = 0; v < 4; ++v) o[u * 4 + v] = w * j[u] * j[v];
    o[16 + u] = w * r * j[u];
  }
  o[20] = r * r;
}

// mode 0: v = (0, 0, src_lambda)
// mode 1: g = fvec_p - kv_p ; rhs = (0, -g, 0) ; grad[b] = g
// mode 2: v = (0, 0, w), w an n_x-vector ; mode 3: out_nx = src[x block]
__global__ void k_adjoint(int mode, int64_t n_x, int64_t n_p, const double* __restrict__ src,
                          const double* __restrict__ fvec, double* __restrict__ out,
                          double* __restrict__ grad) {
  const int b = blockIdx.y;
  const int64_t dim = 2 * n_x + n_p;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < dim; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = (int64_t)b * dim + i;
    const bool in_p = (i >= n_x && i < n_x + n_p);
    if (mode == 0) {
      out[k] = (i >= n_x + n_p) ? src[k] : 0.0;
    } else if (mode == 2) {           // v = (0, 0, w) from an n_x-vector w
      out[k] = (i >= n_x + n_p) ? src[(int64_t)b * n_x + (i - n_x - n_p)] : 0.0;
    } else if (mode == 3) {           // out_nx = x block of src (contiguous n_x per instance)
      if (i < n_x) out[(int64_t)b * n_x + i] = src[k];
    } else if (mode == 4) {           // src = f - K (0, 0, w) evaluated exactly: g = its p block
      if (in_p) {
        const double g = src[k];
        out[k] = -g;
        if (grad) grad[(int64_t)b * n_p + (i - n_x)] = g;
      } else {
        out[k] = 0.0;
      }
    } else {
      if (in_p) {
        const double g = fvec[k] - src[k];
        out[k] = -g;
        if (grad) grad[(int64_t)b * n_p + (i - n_x)] = g;
      } else {
        out[k] = 0.0;
      }
    }
  }
}

// dst[b] = src[b] for instances with mask[b] != 0
__global__ void k_masked_copy(int64_t n, const int32_t* __restrict__ mask, const double* __restrict__ src,
                              double* __restrict__ dst, int64_t stride) {
  const int b = blockIdx.y;
  if (!mask[b]) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[(int64_t)b * stride + i] = src[(int64_t)b * stride + i];
}

}  // namespace

#define VEC_CHECK()                                                                \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      sgn::last_error() = std::string("vector kernel: ") + cudaGetErrorString(_e); \
      return SGN_CUDA_ERROR;                                                       \
    }                                                                              \
  } while (0)

extern "C" {

int sgn_reduce(int32_t op, int64_t n, int32_t batch, const double* d_a, const double* d_b,
               int64_t stride, double* d_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (op) {
    case 0: sgn::count_launch(); k_reduce<0><<<batch, kRed, 0, st>>>(n, d_a, nullptr, stride, d_out); break;
    case 1: sgn::count_launch(); k_reduce<1><<<batch, kRed, 0, st>>>(n, d_a, d_b, stride, d_out); break;
    case 2: sgn::count_launch(); k_reduce<2><<<batch, kRed, 0, st>>>(n, d_a, nullptr, stride, d_out); break;
    default: sgn::last_error() = "bad reduce op"; return SGN_INVALID;
  }
  VEC_CHECK();
  return SGN_OK;
}

int sgn_axpy(int64_t n, int32_t batch, const double* d_alpha, const double* d_x, const double* d_y,
             double* d_out, int64_t stride, void* stream) {
  if (n == 0) return SGN_OK;
  const dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 1024), batch);
  sgn::count_launch();
  k_axpy<<<g, 256, 0, (cudaStream_t)stream>>>(n, d_alpha, d_x, d_y, d_out, stride);
  VEC_CHECK();
  return SGN_OK;
}

// 64-bit fingerprint of each instance's vector: XOR over i of splitmix64(bits(x_i) ^ golden*i)
// (XOR is order-free, so the value is deterministic whatever the block schedule)
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void k_fingerprint(int64_t n, const double* __restrict__ x, int64_t stride,
                              unsigned long long* __restrict__ out) {
  const int b = blockIdx.y;
  unsigned long long h = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    h ^= mix64((unsigned long long)__double_as_longlong(x[(int64_t)b * stride + i]) ^ (0x632be59bd9b4e019ull * (unsigned long long)i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h ^= __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicXor(out + b, h);
}

int sgn_fingerprint(int64_t n, int32_t batch, const double* d_x, int64_t stride, uint64_t* d_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(d_out, 0, (size_t)batch * sizeof(uint64_t), st) != cudaSuccess) {
    sgn::last_error() = "fingerprint memset";
    return SGN_CUDA_ERROR;
  }
  if (n == 0) return SGN_OK;
  const dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 256), batch);
  sgn::count_launch();
  k_fingerprint<<<g, 256, 0, st>>>(n, d_x, stride, reinterpret_cast<unsigned long long*>(d_out));
  VEC_CHECK();
  return SGN_OK;
}

int sgn_masked_copy(int64_t n, int32_t batch, const int32_t* d_mask, const double* d_src,
                    double* d_dst, int64_t stride, void* stream) {
  if (n == 0) return SGN_OK;
  const dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 1024), batch);
  sgn::count_launch();
  k_masked_copy<<<g, 256, 0, (cudaStream_t)stream>>>(n, d_mask, d_src, d_dst, stride);
  VEC_CHECK();
  return SGN_OK;
}

int sgn_lsq_eval(int32_t batch, const sgn_lsq_args* a, const double* d_x, const double* d_p,
                 double* d_vec, double* d_fobj, void* stream) {
  if (!a || !a->part || !a->tickets || batch < 1) { sgn::last_error() = "lsq: bad arguments"; return SGN_INVALID; }
  if (a->rptr && !a->rscr) { sgn::last_error() = "lsq: a residual p-map needs rscr"; return SGN_INVALID; }
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n_x = a->n_x, n_p = a->n_p, nt = a->n_t;
  const int64_t dim = 2 * n_x + n_p;
  if (d_vec && cudaMemsetAsync(d_vec, 0, (size_t)batch * dim * sizeof(double), st) != cudaSuccess) {
    sgn::last_error() = "lsq: vector reset failed";
    return SGN_CUDA_ERROR;
  }
  const int nbt = (int)std::max<int64_t>(1, std::min<int64_t>(kLsqBlocks, (nt + kLsqThreads - 1) / kLsqThreads));
  const int nbp = (int)std::max<int64_t>(1, std::min<int64_t>(kLsqBlocks, (n_p + kLsqThreads - 1) / kLsqThreads));
  sgn::count_launch(2);
  k_lsq_targets<<<dim3(nbt, batch), kLsqThreads, 0, st>>>(n_x, n_p, nt, a->tdofs, a->tvals, a->tstride, a->w_t,
                                                         a->x_scale, d_x, d_p, d_vec, a->rptr, a->ridx, a->rcoef,
                                                         a->rscr, a->part);
  k_lsq_params<<<dim3(nbp, batch), kLsqThreads, 0, st>>>(n_x, n_p, nt, nbt, a->w_reg, d_p, d_vec, d_fobj, a->rtptr,
                                                        a->rtidx, a->rtcoef, a->rscr, a->part, a->tickets);
  VEC_CHECK();
  return SGN_OK;
}

int sgn_restlen_blocks(int64_t ns, int32_t batch, const int32_t* d_conn, const double* d_rest,
                       int64_t rest_stride, const double* d_L0, double w, double* d_out, int64_t out_stride,
                       void* stream) {
  if (ns == 0) return SGN_OK;
  sgn::count_launch();
  k_restlen<<<dim3((unsigned)((ns + 127) / 128), batch), 128, 0, (cudaStream_t)stream>>>(
      ns, d_conn, d_rest, rest_stride, d_L0, w, d_out, out_stride);
  VEC_CHECK();
  return SGN_OK;
}

int sgn_adjoint_step(int32_t mode, int32_t batch, int64_t n_x, int64_t n_p, const double* d_src,
                     const double* d_fvec, double* d_out, double* d_grad, void* stream) {
  const int64_t dim = 2 * n_x + n_p;
  const dim3 g((unsigned)std::min<int64_t>((dim + 255) / 256, 1024), batch);
  sgn::count_launch();
  k_adjoint<<<g, 256, 0, (cudaStream_t)stream>>>(mode, n_x, n_p, d_src, d_fvec, d_out, d_grad);
  VEC_CHECK();
  return SGN_OK;
}

}  // extern "C"
