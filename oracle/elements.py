"""Vectorized NumPy element kernels (oracle; test infrastructure only).

Compressible neo-Hookean simplices (plane-strain triangles, tetrahedra) with a
rest-area/volume-weighted gravity load, and the 2-node spring of the reference
(reference pkg/src/sgnopt/forward.py:29-111).  Energies and gradients are analytic;
second derivatives (d2E/dx2 and the rest-shape mixed block d2E/dx dX) are obtained by
COMPLEX-STEP differentiation of the analytic gradient -- a derivation path
independent of the CUDA kernels (which use closed-form directional derivatives of
the first Piola stress) and exact to machine precision (no subtractive cancellation).

Energy per element (see paper_2107_03285_b200/csrc/elements.cu for the same model):
  E_e = A_e(X) psi(F) + g A_e(X)/nv sum_a x_a[1],
  psi = mu/2 (|F|^2 - d) - mu ln J + lam/2 (ln J)^2,  F = Ds Dm^-1,  A_e = det Dm / d!
"""
from __future__ import annotations

import math

import numpy as np

H_CS = 1e-30  # complex step


def lame(E: float, nu: float) -> tuple[float, float]:
    """(mu, lambda) of isotropic elasticity (3D / plane strain)."""
    return E / (2.0 * (1.0 + nu)), E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))


def _edge(P):
    """Edge matrices D[e] = [P1-P0, P2-P0, ...] as (ne, d, d) with columns = edges."""
    return np.swapaxes(P[:, 1:, :] - P[:, :1, :], 1, 2)


def nh_energy(x, X, mu, lam, g):
    """Per-element energy; x, X: (ne, nv, d)."""
    d = X.shape[2]
    Dm, Ds = _edge(X), _edge(x)
    A = np.linalg.det(Dm) / math.factorial(d)
    F = Ds @ np.linalg.inv(Dm)
    J = np.linalg.det(F)
    lnJ = np.log(J)
    psi = 0.5 * mu * (np.einsum("eij,eij->e", F, F) - d) - mu * lnJ + 0.5 * lam * lnJ ** 2
    return A * psi + g * A / (d + 1) * x[:, :, 1].sum(axis=1)


def _det(M):
    if M.shape[1] == 2:
        return M[:, 0, 0] * M[:, 1, 1] - M[:, 0, 1] * M[:, 1, 0]
    return (M[:, 0, 0] * (M[:, 1, 1] * M[:, 2, 2] - M[:, 1, 2] * M[:, 2, 1])
            - M[:, 0, 1] * (M[:, 1, 0] * M[:, 2, 2] - M[:, 1, 2] * M[:, 2, 0])
            + M[:, 0, 2] * (M[:, 1, 0] * M[:, 2, 1] - M[:, 1, 1] * M[:, 2, 0]))


def _inv(M):
    """Adjugate inverse (works for complex input, unlike LAPACK-free needs)."""
    d = M.shape[1]
    det = _det(M)
    if d == 2:
        adj = np.empty_like(M)
        adj[:, 0, 0] = M[:, 1, 1]; adj[:, 0, 1] = -M[:, 0, 1]
        adj[:, 1, 0] = -M[:, 1, 0]; adj[:, 1, 1] = M[:, 0, 0]
    else:
        adj = np.empty_like(M)
        for i in range(3):
            for j in range(3):
                r = [k for k in range(3) if k != j]
                c = [k for k in range(3) if k != i]
                minor = M[:, r][:, :, c]
                adj[:, i, j] = (-1) ** (i + j) * (minor[:, 0, 0] * minor[:, 1, 1] - minor[:, 0, 1] * minor[:, 1, 0])
    return adj / det[:, None, None]


def nh_grad(x, X, mu, lam, g):
    """dE/dx per element as (ne, nv*d); complex-safe (holomorphic) for complex-step use."""
    ne, nv, d = X.shape
    Dm, Ds = _edge(X), _edge(x)
    B = _inv(Dm)
    A = _det(Dm) / math.factorial(d)
    F = Ds @ B
    J = _det(F)
    FiT = np.swapaxes(_inv(F), 1, 2)
    P = mu * (F - FiT) + lam * np.log(J)[:, None, None] * FiT
    H = A[:, None, None] * (P @ np.swapaxes(B, 1, 2))        # dE/dDs (d x d)
    out = np.zeros((ne, nv, d), dtype=H.dtype)
    out[:, 1:, :] = np.swapaxes(H, 1, 2)
    out[:, 0, :] = -H.sum(axis=2)
    out[:, :, 1] += (g * A / nv)[:, None]
    return out.reshape(ne, nv * d)


def nh_second(x, X, mu, lam, g):
    """(hess, mixed): (ne, nd, nd) each, column k = derivative w.r.t. local dof k."""
    ne, nv, d = X.shape
    nd = nv * d
    hess = np.empty((ne, nd, nd))
    mixed = np.empty((ne, nd, nd))
    xc = x.astype(np.complex128)
    Xc = X.astype(np.complex128)
    for k in range(nd):
        a, i = divmod(k, d)
        xp = xc.copy()
        xp[:, a, i] += 1j * H_CS
        hess[:, :, k] = nh_grad(xp, Xc, mu, lam, g).imag / H_CS
        Xp = Xc.copy()
        Xp[:, a, i] += 1j * H_CS
        mixed[:, :, k] = nh_grad(xc, Xp, mu, lam, g).imag / H_CS
    return hess, mixed


def spring_energy(x, X, k):
    l = np.linalg.norm(x[:, 0] - x[:, 1], axis=1)
    L = np.linalg.norm(X[:, 0] - X[:, 1], axis=1)
    return 0.5 * k * (l - L) ** 2


def spring_grad(x, X, k):
    d = x[:, 0] - x[:, 1]
    l = np.sqrt((d * d).sum(axis=1))
    L = np.sqrt(((X[:, 0] - X[:, 1]) ** 2).sum(axis=1))
    c = k * (l - L) / l
    return np.concatenate([c[:, None] * d, -c[:, None] * d], axis=1)


def spring_second(x, X, k):
    """Spring blocks by complex step on the gradient (same convention as nh_second)."""
    ne, nv, dd = x.shape
    nd = nv * dd
    hess = np.empty((ne, nd, nd))
    mixed = np.empty((ne, nd, nd))
    xc, Xc = x.astype(np.complex128), X.astype(np.complex128)
    for kk in range(nd):
        a, i = divmod(kk, dd)
        xp = xc.copy(); xp[:, a, i] += 1j * H_CS
        hess[:, :, kk] = spring_grad(xp, Xc, k).imag / H_CS
        Xp = Xc.copy(); Xp[:, a, i] += 1j * H_CS
        mixed[:, :, kk] = spring_grad(xc, Xp, k).imag / H_CS
    return hess, mixed
