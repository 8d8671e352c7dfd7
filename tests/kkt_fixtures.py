"""Seeded synthetic KKT systems shared by the CPU and GPU tests (test infrastructure)."""
import numpy as np
import scipy.sparse as sp


def grid_laplacian(nx, ny, dof=1, seed=0):
    """SPD stiffness-like matrix of an nx x ny grid with `dof` unknowns per vertex."""
    rng = np.random.default_rng(seed)
    n = nx * ny
    rows, cols = [], []
    for i in range(nx):
        for j in range(ny):
            v = i * ny + j
            for di, dj in ((1, 0), (0, 1), (1, 1)):
                if i + di < nx and j + dj < ny:
                    u = (i + di) * ny + j + dj
                    rows += [v, u]
                    cols += [u, v]
    a = sp.coo_matrix((-np.ones(len(rows)), (rows, cols)), shape=(n, n)).tocsr()
    a = a + sp.diags(np.asarray(-a.sum(axis=1)).ravel() + 0.1)
    k = sp.kron(a, np.eye(dof) + 0.1 * rng.standard_normal((dof, dof)) * 0).tocsc()
    k = k + sp.diags(rng.uniform(0.0, 0.1, k.shape[0]))
    return sp.csc_matrix(k)


def kkt_system(nx=6, ny=5, dof=2, n_p=7, c_diag=1e-2, seed=0, a_frac=0.3):
    """(K full CSC scipy, n_x, n_p, rhs) with K = [[A,0,G^T],[0,C,Gp^T],[G,Gp,0]]."""
    rng = np.random.default_rng(seed)
    g = grid_laplacian(nx, ny, dof, seed)
    n_x = g.shape[0]
    w = np.where(rng.random(n_x) < a_frac, rng.uniform(0.5, 1.5, n_x), 0.0)
    A = sp.diags(w).tocsc()
    C = sp.diags(np.full(n_p, c_diag)).tocsc() if c_diag else sp.csc_matrix((n_p, n_p))
    gp = sp.random(n_x, n_p, density=min(1.0, 3.0 / n_x), random_state=rng,
                   data_rvs=rng.standard_normal).tocsc()
    for j in range(n_p):  # make every parameter couple to something
        gp[rng.integers(n_x), j] = rng.standard_normal()
    gp = gp.tocsc()
    K = sp.bmat([[A, None, g.T], [None, C, gp.T], [g, gp, None]], format="csc")
    K.sum_duplicates()
    K.sort_indices()
    rhs = np.zeros(2 * n_x + n_p)
    rhs[n_x:n_x + n_p] = rng.standard_normal(n_p)
    return K, n_x, n_p, rhs
