"""NumPy emulation of the device multifrontal LDL^T over an exported assembly tree.

Test infrastructure only: it validates the host symbolic analysis (ordering, front
row structures, extend-add maps) on the CPU, without a GPU, by running the same
front-by-front algorithm densely and checking P^T K P = L D L^T.
"""
import numpy as np


def emulate(K, sym, eps_x=0.0, eps_l=0.0):
    n = K.shape[0]
    perm = sym.perm()
    fr = sym.fronts()
    Kd = K.toarray()[np.ix_(perm, perm)]
    shift = np.zeros(n)
    if sym.n_x > 0:
        u = perm
        shift[u < sym.n_x] = eps_x
        shift[u >= sym.n_x + sym.n_p] = -eps_l
    Ks = Kd + np.diag(shift)
    L = np.eye(n)
    D = np.zeros((n, n))
    upd = {}
    nf = len(fr["first"])
    children = [[] for _ in range(nf)]
    for f in range(nf):
        if fr["parent"][f] >= 0:
            children[fr["parent"][f]].append(f)
    for f in range(nf):
        rows = fr["rows"][fr["rows_ptr"][f]:fr["rows_ptr"][f + 1]]
        first, npiv = int(fr["first"][f]), int(fr["npiv"][f])
        assert np.all(rows[:npiv] == np.arange(first, first + npiv))
        assert np.all(np.diff(rows) > 0)
        nr = len(rows)
        F = np.zeros((nr, nr))
        for lc in range(npiv):
            c = first + lc
            F[lc:, lc] = Ks[rows[lc:], c]
        pos_in = {int(r): i for i, r in enumerate(rows)}
        for ch in children[f]:
            Uc, crows = upd.pop(ch)
            idx = np.array([pos_in[int(r)] for r in crows], dtype=np.int64)
            F[np.ix_(idx, idx)] += np.tril(Uc)
        F = np.tril(F) + np.tril(F, -1).T
        pair = sym.n_x > 0 and np.all(perm[first:first + npiv] < sym.n_x) is False
        unk = perm[rows[:npiv]]
        pair = sym.n_x > 0 and npiv > 0 and not np.all((unk >= sym.n_x) & (unk < sym.n_x + sym.n_p))
        step = 2 if pair else 1
        j = 0
        while j < npiv:
            blk = F[j:j + step, j:j + step].copy()
            inv = np.linalg.inv(blk)
            col = F[j + step:, j:j + step].copy()
            l = col @ inv
            F[j + step:, j + step:] -= l @ col.T
            D[first + j:first + j + step, first + j:first + j + step] = blk
            L[rows[j + step:], first + j:first + j + step] = l
            j += step
        upd[f] = (F[npiv:, npiv:].copy(), rows[npiv:].copy())
    err = np.abs(L @ D @ L.T - Ks).max() / max(np.abs(Ks).max(), 1e-300)
    return L, D, Ks, err, perm
