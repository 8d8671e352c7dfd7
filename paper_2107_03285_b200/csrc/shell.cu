// Discrete-shell element kernels (BASELINE config 4) on B200 (sm_100a).
//
// StVK membrane triangle (plane stress, metric-tensor form) with rest-area-lumped self
// weight, and the Discrete-Shells dihedral hinge energy -- the same model as the CPU oracle
// (oracle/shell.py; no reference implementation exists).  Energies are written
// once as device templates and evaluated on hyper-dual numbers a + b e1 + c e2 + d e1e2: one
// thread per element loops over the (i, j) dof pairs, giving exact d2E/dx2 and rest-shape
// d2E/dx dX entries (no truncation error).  Gradients use the e1 part only.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/sgn_b200.h"
#include "sgn_internal.h"

namespace {

struct HD {
  double a, b, c, d;
};
__device__ __forceinline__ HD hd(double a) { return {a, 0.0, 0.0, 0.0}; }
__device__ __forceinline__ HD operator+(HD x, HD y) { return {x.a + y.a, x.b + y.b, x.c + y.c, x.d + y.d}; }
__device__ __forceinline__ HD operator-(HD x, HD y) { return {x.a - y.a, x.b - y.b, x.c - y.c, x.d - y.d}; }
__device__ __forceinline__ HD operator-(HD x) { return {-x.a, -x.b, -x.c, -x.d}; }
__device__ __forceinline__ HD operator*(HD x, HD y) {
  return {x.a * y.a, x.a * y.b + x.b * y.a, x.a * y.c + x.c * y.a, x.a * y.d + x.b * y.c + x.c * y.b + x.d * y.a};
}
__device__ __forceinline__ HD operator*(double s, HD x) { return {s * x.a, s * x.b, s * x.c, s * x.d}; }
__device__ __forceinline__ HD operator+(HD x, double s) { return {x.a + s, x.b, x.c, x.d}; }
__device__ __forceinline__ HD chain(HD x, double f0, double f1, double f2) {
  return {f0, f1 * x.b, f1 * x.c, f1 * x.d + f2 * x.b * x.c};
}
__device__ __forceinline__ HD recip(HD x) {
  const double r = 1.0 / x.a;
  return chain(x, r, -r * r, 2.0 * r * r * r);
}
__device__ __forceinline__ HD operator/(HD x, HD y) { return x * recip(y); }
__device__ __forceinline__ HD hsqrt(HD x) {
  const double s = sqrt(x.a);
  return chain(x, s, 0.5 / s, -0.25 / (s * x.a));
}
__device__ __forceinline__ HD hatan2(HD y, HD x) {
  const double r2 = x.a * x.a + y.a * y.a, r4 = r2 * r2;
  const double fy = x.a / r2, fx = -y.a / r2;
  const double fyy = -2.0 * x.a * y.a / r4, fxx = 2.0 * x.a * y.a / r4, fxy = (y.a * y.a - x.a * x.a) / r4;
  return {atan2(y.a, x.a), fy * y.b + fx * x.b, fy * y.c + fx * x.c,
          fy * y.d + fx * x.d + fyy * y.b * y.c + fxy * (y.b * x.c + y.c * x.b) + fxx * x.b * x.c};
}

// plain-double rest state (Hessian evaluations: no rest seed, so every rest-only quantity is a
// loop-invariant scalar instead of a hyper-dual with zero dual parts)
__device__ __forceinline__ HD operator*(HD x, double s) { return {s * x.a, s * x.b, s * x.c, s * x.d}; }
__device__ __forceinline__ HD operator-(HD x, double s) { return {x.a - s, x.b, x.c, x.d}; }
__device__ __forceinline__ HD operator-(double s, HD x) { return {s - x.a, -x.b, -x.c, -x.d}; }
__device__ __forceinline__ HD operator/(HD x, double s) { return x * (1.0 / s); }
__device__ __forceinline__ double recip(double x) { return 1.0 / x; }
__device__ __forceinline__ double hsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ double hatan2(double y, double x) { return atan2(y, x); }

template <class T>
struct V3T { T x, y, z; };
typedef V3T<HD> V3;
template <class T>
__device__ __forceinline__ V3T<T> sub(V3T<T> u, V3T<T> v) { return {u.x - v.x, u.y - v.y, u.z - v.z}; }
template <class T>
__device__ __forceinline__ T dot(V3T<T> u, V3T<T> v) { return u.x * v.x + u.y * v.y + u.z * v.z; }
template <class T>
__device__ __forceinline__ V3T<T> cross(V3T<T> u, V3T<T> v) {
  return {u.y * v.z - u.z * v.y, u.z * v.x - u.x * v.z, u.x * v.y - u.y * v.x};
}

// p = (alpha, beta, rho_g, scale, t)
template <class TX>
__device__ __forceinline__ HD membrane_E(const V3* x, const V3T<TX>* X, const double* p) {
  const V3 e1 = sub(x[1], x[0]), e2 = sub(x[2], x[0]);
  const V3T<TX> E1 = sub(X[1], X[0]), E2 = sub(X[2], X[0]);
  const HD a00 = dot(e1, e1), a01 = dot(e1, e2), a11 = dot(e2, e2);
  const TX b00 = dot(E1, E1), b01 = dot(E1, E2), b11 = dot(E2, E2);
  const TX det = b00 * b11 - b01 * b01;
  const TX area = 0.5 * hsqrt(det);
  const TX idet = recip(det);
  const HD m00 = (b11 * a00 - b01 * a01) * idet, m01 = (b11 * a01 - b01 * a11) * idet;
  const HD m10 = (b00 * a01 - b01 * a00) * idet, m11 = (b00 * a11 - b01 * a01) * idet;
  const HD trG = 0.5 * (m00 + m11 + (-2.0));
  const HD d0 = m00 + (-1.0), d1 = m11 + (-1.0);
  const HD trG2 = 0.25 * (d0 * d0 + 2.0 * (m01 * m10) + d1 * d1);
  const HD psi = (0.5 * p[0]) * (trG * trG) + p[1] * trG2;
  const HD zsum = x[0].z + x[1].z + x[2].z;
  return p[4] * (area * psi) + (p[2] * p[4] / 3.0) * (area * zsum);
}

template <class T>
__device__ __forceinline__ T theta(const V3T<T>* x, V3T<T>* n1o, V3T<T>* n2o, V3T<T>* eo) {
  const V3T<T> e = sub(x[1], x[0]);
  const V3T<T> n1 = cross(e, sub(x[2], x[0]));
  const V3T<T> n2 = cross(sub(x[3], x[0]), e);
  const T s = dot(cross(n1, n2), e) / hsqrt(dot(e, e));
  const T c = dot(n1, n2);
  if (n1o) { *n1o = n1; *n2o = n2; *eo = e; }
  return hatan2(s, c);
}

// p = (kb, -, -, scale)
template <class TX>
__device__ __forceinline__ HD hinge_E(const V3* x, const V3T<TX>* X, const double* p) {
  const HD th = theta<HD>(x, nullptr, nullptr, nullptr);
  V3T<TX> n1b, n2b, eb;
  const TX thb = theta<TX>(X, &n1b, &n2b, &eb);
  const TX l2 = dot(eb, eb);
  const TX a1 = 0.5 * hsqrt(dot(n1b, n1b)), a2 = 0.5 * hsqrt(dot(n2b, n2b));
  const HD d = th - thb;
  return p[0] * (d * d) * ((3.0 * l2) / (a1 + a2));
}

template <int NV>
__device__ __forceinline__ HD eval(int kind, const double* xv, const double* Xv, const double* p,
                                   int sx1, int sx2, int sX2) {
  V3 x[NV], X[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    HD c3[3], C3[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int k = v * 3 + i;
      c3[i] = {xv[k], k == sx1 ? 1.0 : 0.0, k == sx2 ? 1.0 : 0.0, 0.0};
      C3[i] = {Xv[k], 0.0, k == sX2 ? 1.0 : 0.0, 0.0};
    }
    x[v] = {c3[0], c3[1], c3[2]};
    X[v] = {C3[0], C3[1], C3[2]};
  }
  return (NV == 3) ? membrane_E<HD>(x, X, p) : hinge_E<HD>(x, X, p);
}

// no rest seed (Hessian / gradient evaluations): the rest state as plain doubles
template <int NV>
__device__ __forceinline__ HD eval_x(const double* xv, const double* Xv, const double* p, int sx1, int sx2) {
  V3 x[NV];
  V3T<double> X[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    HD c3[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int k = v * 3 + i;
      c3[i] = {xv[k], k == sx1 ? 1.0 : 0.0, k == sx2 ? 1.0 : 0.0, 0.0};
    }
    x[v] = {c3[0], c3[1], c3[2]};
    X[v] = {Xv[v * 3], Xv[v * 3 + 1], Xv[v * 3 + 2]};
  }
  return (NV == 3) ? membrane_E<double>(x, X, p) : hinge_E<double>(x, X, p);
}

template <int NV>
__global__ void __launch_bounds__(64)
k_shell_derivs(int64_t ne, const int32_t* __restrict__ conn, const double* __restrict__ pos,
               const double* __restrict__ rest, int64_t vstride, const double* __restrict__ params,
               int64_t pstride, double* __restrict__ hess, double* __restrict__ mixed, int64_t bstride,
               int rmask) {
  constexpr int ND = NV * 3;
  const int b = blockIdx.y;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ne) return;
  double xv[ND], Xv[ND];
  const double* pb = pos + (int64_t)b * vstride;
  const double* rb = rest + (int64_t)b * vstride;
#pragma unroll
  for (int a = 0; a < NV; ++a) {
    const int64_t v = conn[e * NV + a];
#pragma unroll
    for (int i = 0; i < 3; ++i) { xv[a * 3 + i] = pb[v * 3 + i]; Xv[a * 3 + i] = rb[v * 3 + i]; }
  }
  const double* pr = params + (int64_t)b * pstride;
  const double sc = pr[3];
  double* hb = hess + (int64_t)b * bstride + e * ND * ND;
  double* mb = mixed + (int64_t)b * bstride + e * ND * ND;
  for (int i = 0; i < ND; ++i) {
    for (int j = i; j < ND; ++j) {
      const double h = sc * eval_x<NV>(xv, Xv, pr, i, j).d;
      hb[i * ND + j] = h;
      hb[j * ND + i] = h;
    }
    for (int j = 0; j < ND; ++j)        // rest components the p-map never moves are skipped
      if ((rmask >> (j % 3)) & 1) mb[i * ND + j] = sc * eval<NV>(0, xv, Xv, pr, i, -1, j).d;
  }
}

template <int NV>
__global__ void __launch_bounds__(64)
k_shell_energy_grad(int64_t ne, const int32_t* __restrict__ conn, const double* __restrict__ pos,
                    const double* __restrict__ rest, int64_t vstride, const double* __restrict__ params,
                    int64_t pstride, double* __restrict__ energy, double* __restrict__ grad, int64_t bstride) {
  constexpr int ND = NV * 3;
  const int b = blockIdx.y;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ne) return;
  double xv[ND], Xv[ND];
  const double* pb = pos + (int64_t)b * vstride;
  const double* rb = rest + (int64_t)b * vstride;
#pragma unroll
  for (int a = 0; a < NV; ++a) {
    const int64_t v = conn[e * NV + a];
#pragma unroll
    for (int i = 0; i < 3; ++i) { xv[a * 3 + i] = pb[v * 3 + i]; Xv[a * 3 + i] = rb[v * 3 + i]; }
  }
  const double* pr = params + (int64_t)b * pstride;
  const double sc = pr[3];
  double en = 0.0;
  for (int i = 0; i < ND; ++i) {
    const HD E = eval_x<NV>(xv, Xv, pr, i, -1);
    if (grad) grad[(int64_t)b * bstride + e * ND + i] = sc * E.b;
    en = E.a;
  }
  if (energy) energy[(int64_t)b * ne + e] = isfinite(en) ? sc * en : __longlong_as_double(0x7ff8000000000000ll);
}

}  // namespace

namespace sgn {

int launch_shell(bool derivs, int32_t elem_type, int64_t n_elems, int32_t batch, const int32_t* conn,
                 const double* pos, const double* rest, int64_t vstride, const double* params,
                 int64_t pstride, double* out1, double* out2, int64_t bstride, void* stream, int rest_comp_mask) {
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)((n_elems + 63) / 64), batch);
  count_launch();
  if (elem_type == SGN_ELEM_SHELL_MEMBRANE) {
    if (derivs) k_shell_derivs<3><<<grid, 64, 0, st>>>(n_elems, conn, pos, rest, vstride, params, pstride, out1, out2, bstride, rest_comp_mask);
    else k_shell_energy_grad<3><<<grid, 64, 0, st>>>(n_elems, conn, pos, rest, vstride, params, pstride, out1, out2, bstride);
  } else {
    if (derivs) k_shell_derivs<4><<<grid, 64, 0, st>>>(n_elems, conn, pos, rest, vstride, params, pstride, out1, out2, bstride, rest_comp_mask);
    else k_shell_energy_grad<4><<<grid, 64, 0, st>>>(n_elems, conn, pos, rest, vstride, params, pstride, out1, out2, bstride);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { last_error() = std::string("shell kernel: ") + cudaGetErrorString(e); return SGN_CUDA_ERROR; }
  return SGN_OK;
}

}  // namespace sgn
