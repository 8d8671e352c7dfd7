// Element kernels for SGN assembly on B200 (sm_100a).
//
// The reference's only elastic element is the 2-node spring, vectorized in NumPy
// (pkg/src/sgnopt/forward.py:29-111: spring_gradient, spring_hessian_triplets,
// spring_force_rest_jacobian @ spring_length_jacobian).  The BASELINE configs need
// neo-Hookean linear triangles (plane strain) and tetrahedra, which the reference does
// not implement; their CPU restatement lives in oracle/elements.py.
//
// One thread per element; each thread writes its dense element blocks
//   hess [nd x nd] = d2E/dx2          (row-major)
//   mixed[nd x nd] = d2E/dx dX_rest   (row = deformed dof, col = rest dof)
// which the atomic-free gather (k_gather) sums into the KKT CSC pattern in a fixed order.
//
// Energy model (per element e, rest positions X, deformed x):
//   E_e = A_e(X) * psi(F) + g * A_e(X)/nv * sum_a x_a[1]        (nv = nodes per element)
//   psi(F) = mu/2 (tr F^T F - d) - mu ln J + lambda/2 (ln J)^2,  F = Ds Dm^{-1}
// with A_e = det(Dm)/d! (signed measure), g = areal/volumetric load density (downward,
// gravity along -y).  Gradient dE/dx is the equilibrium force residual c(x, p).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/sgn_b200.h"
#include "sgn_internal.h"

namespace {

template <int D>
struct Mat {
  double a[D][D];
};

template <int D>
__device__ __forceinline__ Mat<D> mul(const Mat<D>& x, const Mat<D>& y) {
  Mat<D> r;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += x.a[i][k] * y.a[k][j];
      r.a[i][j] = s;
    }
  return r;
}
template <int D>
__device__ __forceinline__ Mat<D> transpose(const Mat<D>& x) {
  Mat<D> r;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) r.a[i][j] = x.a[j][i];
  return r;
}
__device__ __forceinline__ double det(const Mat<2>& m) { return m.a[0][0] * m.a[1][1] - m.a[0][1] * m.a[1][0]; }
__device__ __forceinline__ double det(const Mat<3>& m) {
  return m.a[0][0] * (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) -
         m.a[0][1] * (m.a[1][0] * m.a[2][2] - m.a[1][2] * m.a[2][0]) +
         m.a[0][2] * (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]);
}
__device__ __forceinline__ Mat<2> inverse(const Mat<2>& m) {
  const double id = 1.0 / det(m);
  Mat<2> r;
  r.a[0][0] = m.a[1][1] * id; r.a[0][1] = -m.a[0][1] * id;
  r.a[1][0] = -m.a[1][0] * id; r.a[1][1] = m.a[0][0] * id;
  return r;
}
__device__ __forceinline__ Mat<3> inverse(const Mat<3>& m) {
  const double id = 1.0 / det(m);
  Mat<3> r;
  r.a[0][0] = (m.a[1][1] * m.a[2][2] - m.a[1][2] * m.a[2][1]) * id;
  r.a[0][1] = (m.a[0][2] * m.a[2][1] - m.a[0][1] * m.a[2][2]) * id;
  r.a[0][2] = (m.a[0][1] * m.a[1][2] - m.a[0][2] * m.a[1][1]) * id;
  r.a[1][0] = (m.a[1][2] * m.a[2][0] - m.a[1][0] * m.a[2][2]) * id;
  r.a[1][1] = (m.a[0][0] * m.a[2][2] - m.a[0][2] * m.a[2][0]) * id;
  r.a[1][2] = (m.a[0][2] * m.a[1][0] - m.a[0][0] * m.a[1][2]) * id;
  r.a[2][0] = (m.a[1][0] * m.a[2][1] - m.a[1][1] * m.a[2][0]) * id;
  r.a[2][1] = (m.a[0][1] * m.a[2][0] - m.a[0][0] * m.a[2][1]) * id;
  r.a[2][2] = (m.a[0][0] * m.a[1][1] - m.a[0][1] * m.a[1][0]) * id;
  return r;
}

// first Piola stress of compressible neo-Hookean and its directional derivative
template <int D>
struct NhState {
  Mat<D> F, FiT;  // F and F^{-T}
  double lnJ;
};
template <int D>
__device__ __forceinline__ Mat<D> nh_P(const NhState<D>& s, double mu, double lam) {
  Mat<D> P;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) P.a[i][j] = mu * (s.F.a[i][j] - s.FiT.a[i][j]) + lam * s.lnJ * s.FiT.a[i][j];
  return P;
}
// dP = mu dF + (mu - lam lnJ) F^{-T} dF^T F^{-T} + lam tr(F^{-1} dF) F^{-T}
template <int D>
__device__ __forceinline__ Mat<D> nh_dP(const NhState<D>& s, const Mat<D>& dF, double mu, double lam) {
  const Mat<D> t1 = mul(mul(s.FiT, transpose(dF)), s.FiT);
  double tr = 0.0;  // tr(F^{-1} dF) = sum_ij FiT_ij dF_ij
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) tr += s.FiT.a[i][j] * dF.a[i][j];
  Mat<D> r;
  const double c = mu - lam * s.lnJ;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) r.a[i][j] = mu * dF.a[i][j] + c * t1.a[i][j] + lam * tr * s.FiT.a[i][j];
  return r;
}

// edge-matrix perturbation for dof (vertex a, axis i): d(D) = e_i e_{a-1}^T (a>0) or -e_i 1^T
template <int D>
__device__ __forceinline__ Mat<D> edge_dir(int a, int i) {
  Mat<D> m;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) m.a[r][c] = 0.0;
  if (a == 0) {
#pragma unroll
    for (int c = 0; c < D; ++c) m.a[i][c] = -1.0;
  } else {
    m.a[i][a - 1] = 1.0;
  }
  return m;
}

// distribute H (d x d, columns = edge vertices 1..d) to the nv*d vertex-dof vector
template <int D>
__device__ __forceinline__ void distribute(const Mat<D>& H, double* out, int stride) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      out[((c + 1) * D + i) * stride] = H.a[i][c];
      s += H.a[i][c];
    }
    out[(0 * D + i) * stride] = -s;
  }
}

template <int D>
__device__ __forceinline__ double factorial_inv() { return D == 2 ? 0.5 : (1.0 / 6.0); }

// Hessian columns (a, 0..D-1) of one neo-Hookean simplex, out[i * ND + r] = d2E/dx_r dx_(a,i)
// (unscaled); the same arithmetic as the column loop of nh_simplex_derivs below.
template <int D>
__device__ __forceinline__ void nh_hess_vertex_cols(const double* xv, const double* Xv, double mu, double lam,
                                                    int a, double sc, double* out) {
  constexpr int ND = (D + 1) * D;
  Mat<D> Ds, Dm;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      Ds.a[i][c] = xv[(c + 1) * D + i] - xv[i];
      Dm.a[i][c] = Xv[(c + 1) * D + i] - Xv[i];
    }
  const Mat<D> B = inverse(Dm);
  const double A = det(Dm) * factorial_inv<D>();
  NhState<D> s;
  s.F = mul(Ds, B);
  const double J = det(s.F);
  s.lnJ = log(J);
  s.FiT = transpose(inverse(s.F));
  const Mat<D> BT = transpose(B);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const Mat<D> dF = mul(edge_dir<D>(a, i), B);
    Mat<D> dH = mul(nh_dP(s, dF, mu, lam), BT);
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) dH.a[r][c] *= A;
    double col[ND];
    distribute(dH, col, 1);
#pragma unroll
    for (int r = 0; r < ND; ++r) out[i * ND + r] = sc * col[r];
  }
}

// neo-Hookean simplex: derivs
template <int D, int LD = (D + 1) * D>
__device__ __forceinline__ void nh_simplex_derivs(const double* xv, const double* Xv, double mu, double lam,
                                                  double gload, double* hess, double* mixed,
                                                  bool want_mixed = true) {
  constexpr int NV = D + 1, ND = NV * D;
  Mat<D> Ds, Dm;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      Ds.a[i][c] = xv[(c + 1) * D + i] - xv[i];
      Dm.a[i][c] = Xv[(c + 1) * D + i] - Xv[i];
    }
  const Mat<D> B = inverse(Dm);
  const double A = det(Dm) * factorial_inv<D>();
  NhState<D> s;
  s.F = mul(Ds, B);
  const double J = det(s.F);
  s.lnJ = log(J);
  s.FiT = transpose(inverse(s.F));
  const Mat<D> P = nh_P(s, mu, lam);
  const Mat<D> BT = transpose(B);
  const Mat<D> PBT = mul(P, BT);
  // hessian columns: perturb deformed dof (a, i); triangles unroll fully (static staging
  // indices), tets keep the vertex loop (their staging is shared memory: dynamic is fine)
#pragma unroll (D == 2 ? NV : 1)
  for (int a = 0; a < NV; ++a)
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int col = a * D + i;
      const Mat<D> dF = mul(edge_dir<D>(a, i), B);
      Mat<D> dH = mul(nh_dP(s, dF, mu, lam), BT);
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) dH.a[r][c] *= A;
      distribute(dH, hess + col, ND);
    }
  if (!want_mixed) return;
  // mixed columns: perturb rest dof (a, i)
#pragma unroll (D == 2 ? NV : 1)
  for (int a = 0; a < NV; ++a)
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int col = a * D + i;
      const Mat<D> dDm = edge_dir<D>(a, i);
      const Mat<D> dDmB = mul(dDm, B);
      double trBdDm = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) trBdDm += mul(B, dDm).a[k][k];
      const double dA = A * trBdDm;
      Mat<D> dF = mul(s.F, dDmB);
      Mat<D> dB = mul(B, dDmB);  // dB = -B dDm B
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) { dF.a[r][c] = -dF.a[r][c]; dB.a[r][c] = -dB.a[r][c]; }
      const Mat<D> t2 = mul(nh_dP(s, dF, mu, lam), BT);
      const Mat<D> t3 = mul(P, transpose(dB));
      Mat<D> dH;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) dH.a[r][c] = dA * PBT.a[r][c] + A * (t2.a[r][c] + t3.a[r][c]);
      distribute(dH, mixed + col, ND);
      // gravity load: d2/dy_a dX = g/NV * dA on every vertex's axis-1 row
#pragma unroll
      for (int v = 0; v < NV; ++v) mixed[(v * D + 1) * ND + col] += gload * dA / NV;
    }
}

template <int D>
__device__ void nh_simplex_energy_grad(const double* xv, const double* Xv, double mu, double lam,
                                       double gload, double* energy, double* grad) {
  constexpr int NV = D + 1;
  Mat<D> Ds, Dm;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      Ds.a[i][c] = xv[(c + 1) * D + i] - xv[i];
      Dm.a[i][c] = Xv[(c + 1) * D + i] - Xv[i];
    }
  const Mat<D> B = inverse(Dm);
  const double A = det(Dm) * factorial_inv<D>();
  NhState<D> s;
  s.F = mul(Ds, B);
  const double J = det(s.F);
  s.lnJ = log(J);
  double I1 = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) I1 += s.F.a[i][j] * s.F.a[i][j];
  const double psi = 0.5 * mu * (I1 - D) - mu * s.lnJ + 0.5 * lam * s.lnJ * s.lnJ;
  double ysum = 0.0;
#pragma unroll
  for (int v = 0; v < NV; ++v) ysum += xv[v * D + 1];
  *energy = (J > 0.0) ? A * psi + gload * A / NV * ysum : __longlong_as_double(0x7ff8000000000000ll);
  s.FiT = transpose(inverse(s.F));
  Mat<D> H = mul(nh_P(s, mu, lam), transpose(B));
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) H.a[r][c] *= A;
  distribute(H, grad, 1);
#pragma unroll
  for (int v = 0; v < NV; ++v) grad[v * D + 1] += gload * A / NV;
}

// spring (any dim): E = k/2 (l - L)^2, L = |X_a - X_b|
template <int D>
__device__ void spring_derivs(const double* xv, const double* Xv, double k, double* hess, double* mixed) {
  constexpr int ND = 2 * D;
  double d[D], Dr[D], l2 = 0.0, L2 = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    d[i] = xv[i] - xv[D + i];
    Dr[i] = Xv[i] - Xv[D + i];
    l2 += d[i] * d[i];
    L2 += Dr[i] * Dr[i];
  }
  const double l = sqrt(l2), L = sqrt(L2);
  const double coef = (l - L) / l;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double oo = (d[i] / l) * (d[j] / l);
      const double h = k * (oo + coef * ((i == j ? 1.0 : 0.0) - oo));
      hess[i * ND + j] = h;
      hess[(D + i) * ND + D + j] = h;
      hess[i * ND + D + j] = -h;
      hess[(D + i) * ND + j] = -h;
      const double m = -k * (d[i] / l) * (Dr[j] / L);
      mixed[i * ND + j] = m;
      mixed[(D + i) * ND + D + j] = m;
      mixed[i * ND + D + j] = -m;
      mixed[(D + i) * ND + j] = -m;
    }
}

template <int D>
__device__ void spring_energy_grad(const double* xv, const double* Xv, double k, double* energy, double* grad) {
  double d[D], l2 = 0.0, L2 = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    d[i] = xv[i] - xv[D + i];
    const double r = Xv[i] - Xv[D + i];
    l2 += d[i] * d[i];
    L2 += r * r;
  }
  const double l = sqrt(l2), L = sqrt(L2);
  *energy = 0.5 * k * (l - L) * (l - L);
  const double c = k * (l - L) / l;
#pragma unroll
  for (int i = 0; i < D; ++i) { grad[i] = c * d[i]; grad[D + i] = -c * d[i]; }
}

// params layout per instance: [mu, lambda, gload, scale, k_0, k_1, ...]; outputs are multiplied
// by `scale` (the 1/E equilibrium-row scaling); springs read per-element k_e
template <int TYPE, int D>
__global__ void k_elem_derivs(int64_t ne, const int32_t* __restrict__ conn, const double* __restrict__ pos,
                              const double* __restrict__ rest, int64_t vstride,
                              const double* __restrict__ params, int64_t pstride,
                              double* __restrict__ hess, double* __restrict__ mixed, int64_t bstride) {
  constexpr int NV = (TYPE == SGN_ELEM_SPRING) ? 2 : D + 1;
  constexpr int ND = NV * D;
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
    for (int i = 0; i < D; ++i) { xv[a * D + i] = pb[v * D + i]; Xv[a * D + i] = rb[v * D + i]; }
  }
  double h[ND * ND], m[ND * ND];
  const double* pr = params + (int64_t)b * pstride;
  if (TYPE == SGN_ELEM_SPRING) spring_derivs<D>(xv, Xv, pr[4 + e], h, m);
  else nh_simplex_derivs<D>(xv, Xv, pr[0], pr[1], pr[2], h, m);
  const double sc = pr[3];
  double* hb = hess + (int64_t)b * bstride + e * ND * ND;
  double* mb = mixed + (int64_t)b * bstride + e * ND * ND;
#pragma unroll
  for (int k = 0; k < ND * ND; ++k) { hb[k] = sc * h[k]; mb[k] = sc * m[k]; }
}

template <int TYPE, int D>
__global__ void k_elem_energy_grad(int64_t ne, const int32_t* __restrict__ conn, const double* __restrict__ pos,
                                   const double* __restrict__ rest, int64_t vstride,
                                   const double* __restrict__ params, int64_t pstride,
                                   double* __restrict__ energy, double* __restrict__ grad, int64_t bstride) {
  constexpr int NV = (TYPE == SGN_ELEM_SPRING) ? 2 : D + 1;
  constexpr int ND = NV * D;
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
    for (int i = 0; i < D; ++i) { xv[a * D + i] = pb[v * D + i]; Xv[a * D + i] = rb[v * D + i]; }
  }
  double en, g[ND];
  const double* pr = params + (int64_t)b * pstride;
  if (TYPE == SGN_ELEM_SPRING) spring_energy_grad<D>(xv, Xv, pr[4 + e], &en, g);
  else nh_simplex_energy_grad<D>(xv, Xv, pr[0], pr[1], pr[2], &en, g);
  const double sc = pr[3];
  if (energy) energy[(int64_t)b * ne + e] = sc * en;
  if (grad) {
    double* gb = grad + (int64_t)b * bstride + e * ND;
#pragma unroll
    for (int k = 0; k < ND; ++k) gb[k] = sc * g[k];
  }
}

// Neo-Hookean simplices (assembly throughput path): one thread per element, all columns
// unrolled, blocks staged in shared memory (element stride ND*ND+1 doubles: odd, so the
// per-thread staging stores are bank-conflict free), then copied out by the whole CTA as
// one contiguous, coalesced run of [hess | mixed] rows per block (the per-thread stores of
// the register/local-memory variant touched one sector per element and entry).
template <int D, int EPB>
__global__ void __launch_bounds__(EPB)
k_nh_derivs(int64_t ne, const int32_t* __restrict__ conn, const double* __restrict__ pos,
            const double* __restrict__ rest, int64_t vstride, const double* __restrict__ params,
            int64_t pstride, double* __restrict__ hess, double* __restrict__ mixed,
            const int32_t* __restrict__ mslot, const int32_t* __restrict__ elist, int64_t bstride) {
  constexpr int NV = D + 1, ND = NV * D, NN = ND * ND, SS = NN + 1;
  extern __shared__ double stage[];             // [EPB][SS] hess, then [EPB][SS] mixed
  const int b = blockIdx.y;
  const int64_t e0 = (int64_t)blockIdx.x * EPB;
  // elist (mixed-only mode): entry t is element elist[t], its mixed block goes to slot t
  const int64_t e = (elist && e0 + threadIdx.x < ne) ? (int64_t)__ldg(elist + e0 + threadIdx.x) : e0 + threadIdx.x;
  const double* pr = params + (int64_t)b * pstride;
  const double sc = pr[3];
  const bool in_range = e0 + threadIdx.x < ne;
  const bool want_mixed = in_range && mixed && (elist || !mslot || mslot[e] >= 0);
  if (in_range && (hess || want_mixed)) {
    double xv[ND], Xv[ND];
    const double* pb = pos + (int64_t)b * vstride;
    const double* rb = rest + (int64_t)b * vstride;
    int32_t vv[NV];
#pragma unroll
    for (int a = 0; a < NV; ++a) vv[a] = __ldg(conn + e * NV + a);
#pragma unroll
    for (int a = 0; a < NV; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) { xv[a * D + i] = pb[(int64_t)vv[a] * D + i]; Xv[a * D + i] = rb[(int64_t)vv[a] * D + i]; }
    double* hs = stage + threadIdx.x * SS;
    double* ms = stage + (EPB + threadIdx.x) * SS;
    nh_simplex_derivs<D>(xv, Xv, pr[0], pr[1], pr[2], hs, ms, want_mixed);
#pragma unroll
    for (int k = 0; k < NN; ++k) hs[k] *= sc;
    if (want_mixed)
#pragma unroll
      for (int k = 0; k < NN; ++k) ms[k] *= sc;
  }
  __syncthreads();
  const int nel = (int)(ne - e0 < EPB ? ne - e0 : EPB);
  const int64_t nloc = (int64_t)nel * NN;
  if (hess) {
    double* hb = hess + (int64_t)b * bstride + e0 * NN;
    for (int64_t f = threadIdx.x; f < nloc; f += EPB) {
      const int j = (int)(f / NN), k = (int)(f - (int64_t)j * NN);
      hb[f] = stage[j * SS + k];
    }
  }
  if (!mixed) return;
  // compact slots are increasing in e, so the block's support elements are one contiguous run
  double* mb = mixed + (int64_t)b * bstride;
  for (int64_t f = threadIdx.x; f < nloc; f += EPB) {
    const int j = (int)(f / NN), k = (int)(f - (int64_t)j * NN);
    const int64_t slot = (mslot && !elist) ? (int64_t)__ldg(mslot + e0 + j) : e0 + j;
    if (slot >= 0) mb[slot * NN + k] = stage[(EPB + j) * SS + k];
  }
}

template <int D, int EPB>
int launch_nh_derivs(int64_t ne, int32_t batch, const int32_t* conn, const double* pos, const double* rest,
                     int64_t vstride, const double* params, int64_t pstride, double* hess, double* mixed,
                     const int32_t* mslot, const int32_t* elist, int64_t bstride, cudaStream_t st) {
  constexpr int ND = (D + 1) * D;
  const size_t smem = 2 * EPB * (ND * ND + 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k_nh_derivs<D, EPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SGN_CUDA_ERROR;
    attr = true;
  }
  const dim3 grid((unsigned)((ne + EPB - 1) / EPB), batch);
  k_nh_derivs<D, EPB><<<grid, EPB, smem, st>>>(ne, conn, pos, rest, vstride, params, pstride, hess, mixed, mslot,
                                                elist, bstride);
  return SGN_OK;
}

// Fused vertex-centric G_x assembly (engine.VertexPlan): a group of GS lanes per vertex
// task; lane s computes the Hessian columns of the task vertex in its incident element s
// (ascending element order) into shared memory; then each output -- column dof (v, i),
// row dof r -- is the fixed-order sum of its staged element entries, written to
// K[lambda_r, x_c], K[x_c, lambda_r] (kv) and G_x[r, c] (gv; either may be NULL).
template <int GS>
constexpr int vertex_gpb() { return GS == 6 ? 16 : 128 / GS; }   // groups per block

template <int D, int GS>
__global__ void __launch_bounds__(vertex_gpb<GS>() * GS)
k_vertex_assemble(int32_t ntask, const int32_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc_ea,
                  const int32_t* __restrict__ out_ptr, const int32_t* __restrict__ out_dst,
                  const int32_t* __restrict__ con_ptr, const int32_t* __restrict__ con_idx,
                  const int32_t* __restrict__ conn, const double* __restrict__ pos,
                  const double* __restrict__ rest, int64_t vstride, const double* __restrict__ params,
                  int64_t pstride, double* __restrict__ kv, int64_t kstride, double* __restrict__ gv,
                  int64_t gstride) {
  constexpr int NV = D + 1, ND = NV * D, SLOT = D * ND, GPB = vertex_gpb<GS>();
  __shared__ double sm[GPB][GS * SLOT];
  const int grp = threadIdx.x / GS, lane = threadIdx.x % GS;
  const int64_t task = (int64_t)blockIdx.x * GPB + grp;
  const int b = blockIdx.y;
  const double* pr = params + (int64_t)b * pstride;
  if (task < ntask) {
    const int i0 = __ldg(inc_ptr + task), n = __ldg(inc_ptr + task + 1) - i0;
    if (lane < n) {
      const int ea = __ldg(inc_ea + i0 + lane);
      const int64_t e = ea >> 2;
      const int a = ea & 3;
      const double* pb = pos + (int64_t)b * vstride;
      const double* rb = rest + (int64_t)b * vstride;
      double xv[ND], Xv[ND];
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int64_t v = __ldg(conn + e * NV + q);
#pragma unroll
        for (int i = 0; i < D; ++i) { xv[q * D + i] = pb[v * D + i]; Xv[q * D + i] = rb[v * D + i]; }
      }
      nh_hess_vertex_cols<D>(xv, Xv, pr[0], pr[1], a, pr[3], &sm[grp][lane * SLOT]);
    }
  }
  __syncthreads();
  if (task >= ntask) return;
  const int o0 = __ldg(out_ptr + task), o1 = __ldg(out_ptr + task + 1);
  double* kb = kv ? kv + (int64_t)b * kstride : nullptr;
  double* gb = gv ? gv + (int64_t)b * gstride : nullptr;
  for (int o = o0 + lane; o < o1; o += GS) {
    double v = 0.0;
    const int t1 = __ldg(con_ptr + o + 1);
    for (int t = __ldg(con_ptr + o); t < t1; ++t) v += sm[grp][__ldg(con_idx + t)];
    if (kb) {
      kb[__ldg(out_dst + 3 * o)] = v;
      kb[__ldg(out_dst + 3 * o + 1)] = v;
    }
    if (gb) gb[__ldg(out_dst + 3 * o + 2)] = v;
  }
}

template <int D, int GS>
void launch_vertex(int32_t ntask, int32_t batch, const int32_t* inc_ptr, const int32_t* inc_ea,
                   const int32_t* out_ptr, const int32_t* out_dst, const int32_t* con_ptr,
                   const int32_t* con_idx, const int32_t* conn, const double* pos, const double* rest,
                   int64_t vstride, const double* params, int64_t pstride, double* kv, int64_t kstride,
                   double* gv, int64_t gstride, cudaStream_t st) {
  constexpr int GPB = vertex_gpb<GS>();
  const dim3 grid((unsigned)((ntask + GPB - 1) / GPB), batch);
  k_vertex_assemble<D, GS><<<grid, GPB * GS, 0, st>>>(ntask, inc_ptr, inc_ea, out_ptr, out_dst, con_ptr, con_idx,
                                                  conn, pos, rest, vstride, params, pstride, kv, kstride, gv,
                                                  gstride);
}

// out[dst[k]] = base[k] + sum coef * buf[idx]  (the gather restricted to a list of outputs)
__global__ void k_gather_to(int64_t n_out, const int64_t* __restrict__ dst, const double* __restrict__ base,
                            const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                            const double* __restrict__ coef, const double* __restrict__ buf,
                            int64_t buf_stride, double* __restrict__ out, int64_t out_stride) {
  const int b = blockIdx.y;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_out) return;
  const double* bb = buf + (int64_t)b * buf_stride;
  double s = base ? base[k] : 0.0;
  const int64_t e = ptr[k + 1];
  for (int64_t t = ptr[k]; t < e; ++t) s += (coef ? coef[t] : 1.0) * bb[idx[t]];
  out[(int64_t)b * out_stride + dst[k]] = s;
}

__global__ void k_gather(int64_t n_out, const double* __restrict__ base, int64_t base_stride,
                         const int64_t* __restrict__ ptr, const int64_t* __restrict__ idx,
                         const double* __restrict__ coef, const double* __restrict__ buf,
                         int64_t buf_stride, double* __restrict__ out, int64_t out_stride) {
  const int b = blockIdx.y;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n_out) return;
  const double* bb = buf + (int64_t)b * buf_stride;
  double s = base ? base[(int64_t)b * base_stride + k] : 0.0;
  const int64_t e = ptr[k + 1];
  for (int64_t t = ptr[k]; t < e; ++t) s += (coef ? coef[t] : 1.0) * bb[idx[t]];
  out[(int64_t)b * out_stride + k] = s;
}

}  // namespace

#define ELEM_CHECK()                                                               \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) {                                                       \
      sgn::last_error() = std::string("element kernel: ") + cudaGetErrorString(_e); \
      return SGN_CUDA_ERROR;                                                       \
    }                                                                              \
  } while (0)

extern "C" {

// spring_dim: for SGN_ELEM_SPRING the spatial dimension is params[3] of instance 0 is not
// read on the host; springs are dispatched by elem_type + 100*dim (2 or 3).
int sgn_element_derivs(int32_t elem_type, int64_t n_elems, int32_t batch, const int32_t* d_conn,
                       const double* d_pos, const double* d_rest, int64_t vert_stride,
                       const double* d_params, int64_t param_stride, double* d_hess,
                       double* d_mixed, const int32_t* d_mslot, int64_t buf_stride, void* stream) {
  return sgn_element_derivs_ex(elem_type, n_elems, batch, d_conn, d_pos, d_rest, vert_stride, d_params,
                               param_stride, d_hess, d_mixed, d_mslot, buf_stride, 7, stream);
}

int sgn_element_derivs_ex(int32_t elem_type, int64_t n_elems, int32_t batch, const int32_t* d_conn,
                          const double* d_pos, const double* d_rest, int64_t vert_stride,
                          const double* d_params, int64_t param_stride, double* d_hess,
                          double* d_mixed, const int32_t* d_mslot, int64_t buf_stride,
                          int32_t rest_comp_mask, void* stream) {
  if (d_mslot && elem_type != SGN_ELEM_NH_TRI && elem_type != SGN_ELEM_NH_TET) {
    sgn::last_error() = "mixed slots are supported for neo-Hookean simplices only";
    return SGN_INVALID;
  }
  // non-simplex kinds always write every mixed block; a NULL d_mixed goes to scratch-free
  // Hessian-only paths for simplices, and is rejected for the others
  if ((!d_mixed || !d_hess) && elem_type != SGN_ELEM_NH_TRI && elem_type != SGN_ELEM_NH_TET) {
    sgn::last_error() = "Hessian-only evaluation is supported for neo-Hookean simplices only";
    return SGN_INVALID;
  }
  if (n_elems == 0) return SGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)((n_elems + 127) / 128), batch);
  const dim3 grid64((unsigned)((n_elems + 63) / 64), batch);   // tets: 64-thread blocks
  switch (elem_type) {
    case SGN_ELEM_SPRING:
    case SGN_ELEM_SPRING + 200:
      sgn::count_launch();
      k_elem_derivs<SGN_ELEM_SPRING, 2><<<grid, 128, 0, st>>>(n_elems, d_conn, d_pos, d_rest, vert_stride,
                                                              d_params, param_stride, d_hess, d_mixed, buf_stride);
      break;
    case SGN_ELEM_SPRING + 300:
      sgn::count_launch();
      k_elem_derivs<SGN_ELEM_SPRING, 3><<<grid, 128, 0, st>>>(n_elems, d_conn, d_pos, d_rest, vert_stride,
                                                              d_params, param_stride, d_hess, d_mixed, buf_stride);
      break;
    case SGN_ELEM_NH_TRI:
      sgn::count_launch();
      if (launch_nh_derivs<2, 64>(n_elems, batch, d_conn, d_pos, d_rest, vert_stride, d_params, param_stride,
                                  d_hess, d_mixed, d_mslot, nullptr, buf_stride, st) != SGN_OK) {
        sgn::last_error() = "k_nh_derivs<2>: smem attribute";
        return SGN_CUDA_ERROR;
      }
      break;
    case SGN_ELEM_NH_TET:
      sgn::count_launch();
      if (launch_nh_derivs<3, 32>(n_elems, batch, d_conn, d_pos, d_rest, vert_stride, d_params, param_stride,
                                  d_hess, d_mixed, d_mslot, nullptr, buf_stride, st) != SGN_OK) {
        sgn::last_error() = "k_nh_derivs<3>: smem attribute";
        return SGN_CUDA_ERROR;
      }
      break;
    case SGN_ELEM_SHELL_MEMBRANE:
    case SGN_ELEM_HINGE:
      return sgn::launch_shell(true, elem_type, n_elems, batch, d_conn, d_pos, d_rest, vert_stride,
                               d_params, param_stride, d_hess, d_mixed, buf_stride, stream, rest_comp_mask);
    default:
      sgn::last_error() = "unknown element type";
      return SGN_INVALID;
  }
  ELEM_CHECK();
  return SGN_OK;
}

int sgn_element_energy_grad(int32_t elem_type, int64_t n_elems, int32_t batch, const int32_t* d_conn,
                            const double* d_pos, const double* d_rest, int64_t vert_stride,
                            const double* d_params, int64_t param_stride, double* d_energy,
                            double* d_grad, int64_t buf_stride, void* stream) {
  if (n_elems == 0) return SGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)((n_elems + 127) / 128), batch);
  const dim3 grid64((unsigned)((n_elems + 63) / 64), batch);   // tets: 64-thread blocks
  switch (elem_type) {
    case SGN_ELEM_SPRING:
    case SGN_ELEM_SPRING + 200:
      sgn::count_launch();
      k_elem_energy_grad<SGN_ELEM_SPRING, 2><<<grid, 128, 0, st>>>(n_elems, d_conn, d_pos, d_rest, vert_stride,
                                                                   d_params, param_stride, d_energy, d_grad, buf_stride);
      break;
    case SGN_ELEM_SPRING + 300:
      sgn::count_launch();
      k_elem_energy_grad<SGN_ELEM_SPRING, 3><<<grid, 128, 0, st>>>(n_elems, d_conn, d_pos, d_rest, vert_stride,
                                                                   d_params, param_stride, d_energy, d_grad, buf_stride);
      break;
    case SGN_ELEM_NH_TRI:
      sgn::count_launch();
      k_elem_energy_grad<SGN_ELEM_NH_TRI, 2><<<grid, 128, 0, st>>>(n_elems, d_conn, d_pos, d_rest, vert_stride,
                                                                   d_params, param_stride, d_energy, d_grad, buf_stride);
      break;
    case SGN_ELEM_NH_TET:
      sgn::count_launch();
      k_elem_energy_grad<SGN_ELEM_NH_TET, 3><<<grid64, 64, 0, st>>>(n_elems, d_conn, d_pos, d_rest, vert_stride,
                                                                  d_params, param_stride, d_energy, d_grad, buf_stride);
      break;
    case SGN_ELEM_SHELL_MEMBRANE:
    case SGN_ELEM_HINGE:
      return sgn::launch_shell(false, elem_type, n_elems, batch, d_conn, d_pos, d_rest, vert_stride,
                               d_params, param_stride, d_energy, d_grad, buf_stride, stream);
    default:
      sgn::last_error() = "unknown element type";
      return SGN_INVALID;
  }
  ELEM_CHECK();
  return SGN_OK;
}

int sgn_element_mixed(int32_t elem_type, int64_t n_list, int32_t batch, const int32_t* d_elems,
                      const int32_t* d_conn, const double* d_pos, const double* d_rest, int64_t vert_stride,
                      const double* d_params, int64_t param_stride, double* d_mixed, int64_t buf_stride,
                      void* stream) {
  if (n_list == 0) return SGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (elem_type == SGN_ELEM_NH_TRI)
    rc = launch_nh_derivs<2, 64>(n_list, batch, d_conn, d_pos, d_rest, vert_stride, d_params, param_stride,
                                 nullptr, d_mixed, nullptr, d_elems, buf_stride, st);
  else if (elem_type == SGN_ELEM_NH_TET)
    rc = launch_nh_derivs<3, 32>(n_list, batch, d_conn, d_pos, d_rest, vert_stride, d_params, param_stride,
                                 nullptr, d_mixed, nullptr, d_elems, buf_stride, st);
  else {
    sgn::last_error() = "sgn_element_mixed: neo-Hookean simplices only";
    return SGN_INVALID;
  }
  if (rc != SGN_OK) { sgn::last_error() = "k_nh_derivs: smem attribute"; return rc; }
  sgn::count_launch();
  ELEM_CHECK();
  return SGN_OK;
}

int sgn_vertex_assemble(int32_t elem_type, int32_t n_task, int32_t group, int32_t batch,
                        const int32_t* d_inc_ptr, const int32_t* d_inc_ea, const int32_t* d_out_ptr,
                        const int32_t* d_out_dst, const int32_t* d_con_ptr, const int32_t* d_con_idx,
                        const int32_t* d_conn, const double* d_pos, const double* d_rest, int64_t vert_stride,
                        const double* d_params, int64_t param_stride, double* d_kvals, int64_t kstride,
                        double* d_gvals, int64_t gstride, void* stream) {
  if (n_task == 0) return SGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
#define VA_ARGS n_task, batch, d_inc_ptr, d_inc_ea, d_out_ptr, d_out_dst, d_con_ptr, d_con_idx, d_conn, d_pos, \
                d_rest, vert_stride, d_params, param_stride, d_kvals, kstride, d_gvals, gstride, st
  if (elem_type == SGN_ELEM_NH_TRI && group <= 6) launch_vertex<2, 6>(VA_ARGS);
  else if (elem_type == SGN_ELEM_NH_TRI && group <= 8) launch_vertex<2, 8>(VA_ARGS);
  else if (elem_type == SGN_ELEM_NH_TRI && group <= 16) launch_vertex<2, 16>(VA_ARGS);
  else if (elem_type == SGN_ELEM_NH_TET && group <= 16) launch_vertex<3, 16>(VA_ARGS);
  else if (elem_type == SGN_ELEM_NH_TET && group <= 32) launch_vertex<3, 32>(VA_ARGS);
  else {
    sgn::last_error() = "vertex assembly: unsupported element type / incidence";
    return SGN_INVALID;
  }
#undef VA_ARGS
  sgn::count_launch();
  ELEM_CHECK();
  return SGN_OK;
}

int sgn_gather_to(int64_t n_out, int32_t batch, const int64_t* d_dst, const double* d_base,
                  const int64_t* d_ptr, const int64_t* d_idx, const double* d_coef, const double* d_buf,
                  int64_t buf_stride, double* d_out, int64_t out_stride, void* stream) {
  if (n_out == 0) return SGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)((n_out + 255) / 256), batch);
  sgn::count_launch();
  k_gather_to<<<grid, 256, 0, st>>>(n_out, d_dst, d_base, d_ptr, d_idx, d_coef, d_buf, buf_stride, d_out,
                                    out_stride);
  ELEM_CHECK();
  return SGN_OK;
}

int sgn_gather_values(int64_t n_out, int32_t batch, const double* d_base, int64_t base_stride,
                      const int64_t* d_ptr, const int64_t* d_idx, const double* d_coef,
                      const double* d_buf, int64_t buf_stride, double* d_out, int64_t out_stride,
                      void* stream) {
  if (n_out == 0) return SGN_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)((n_out + 255) / 256), batch);
  sgn::count_launch();
  k_gather<<<grid, 256, 0, st>>>(n_out, d_base, base_stride, d_ptr, d_idx, d_coef, d_buf, buf_stride,
                                 d_out, out_stride);
  ELEM_CHECK();
  return SGN_OK;
}

}  // extern "C"
