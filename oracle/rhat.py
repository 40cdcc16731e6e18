"""Observation-error (and D) approximations as dense matrices (ORACLE, tests only).

  R_diag   P:L415: the diagonal of R_i.
  R_block  Algorithm 1: first-super-diagonal block norms
           normvec(j) = ||R(pst(j):pst(j+1)-1, pst(j+1):pst(j+2)-1)||_F / sqrt(pvec_j pvec_{j+1});
           where normvec(j) < tol the whole coupling across the cut pst(j+1) is
           zeroed.  maxsize / numproc adjustments are applied only when given
           (reading A7: uniform pvec, tol = +inf, i.e. every cut applied).
  R_RR     Algorithm 2: R_i + gamma I; gamma = lambda_min(R_i)
           online unless given (reading A5).
  R_ME     Algorithm 3: eigenvalues <= T raised to T.  Online T
            = the smallest eigenvalue strictly above lambda_min
           (relative gap 1e-10; reading A6).
  D_hat    P:L572: ridge B + delta I, Q + delta I (delta = 0.01 in the paper);
           default D_hat = D (reading A4).
Every function returns the dense matrix of the definition (R_ME by its
eigendecomposition, no Woodbury).  The oracle applies their inverses with LAPACK
Cholesky solves against these matrices (oracle/saddle.py: scipy cho_factor once per
distinct block, cho_solve per window -- the paper applies R_hat^{-1} "using the
Cholesky factors", and D_hat^{-1} by its factors); the explicit
route (oracle/saddle.py explicit_apply_Pinv) is an LU solve with the assembled P.
Both are independent of the CUDA path's factorisations and kernels.
"""
import numpy as np

REL_GAP = 1e-10


def r_diag(R):
    return np.diag(np.diag(R))


def block_starts(pvec):
    return np.concatenate([[0], np.cumsum(pvec)]).astype(int)


def r_block(R, pvec, tol=np.inf, maxsize=None, numproc=None):
    """Algorithm 1.  Returns (R_block, list of (start, end) diagonal blocks)."""
    pvec = [int(v) for v in pvec]
    p = int(sum(pvec))
    assert p == R.shape[0]
    pn = len(pvec)
    pst = block_starts(pvec)
    Rb = R.copy()
    normvec = []
    for j in range(pn - 1):
        blk = R[pst[j]:pst[j + 1], pst[j + 1]:pst[j + 2]]
        normvec.append(np.linalg.norm(blk, "fro") / np.sqrt(pvec[j] * pvec[j + 1]))
    cuts = []
    for j in range(pn - 1):
        if normvec[j] < tol:
            c = pst[j + 1]
            Rb[c:p, 0:c] = 0.0
            Rb[0:c, c:p] = 0.0
            cuts.append(c)
    blocks = []
    edges = [0] + cuts + [p]
    for a, b in zip(edges[:-1], edges[1:]):
        blocks.append((a, b))
    if maxsize is not None:
        sizes = [b - a for a, b in blocks]
        i = int(np.argmax(sizes))
        if sizes[i] > maxsize:
            a, b = blocks[i]
            mid = a + (b - a + 1) // 2
            Rb[mid:b, a:mid] = 0.0
            Rb[a:mid, mid:b] = 0.0
            blocks[i:i + 1] = [(a, mid), (mid, b)]
    if numproc is not None:
        if len(blocks) > numproc:
            sums = [(blocks[i][1] - blocks[i][0]) + (blocks[i + 1][1] - blocks[i + 1][0])
                    for i in range(len(blocks) - 1)]
            i = int(np.argmin(sums))
            a, b = blocks[i][0], blocks[i + 1][1]
            Rb[a:b, a:b] = R[a:b, a:b]
            blocks[i:i + 2] = [(a, b)]
        elif len(blocks) < numproc - 2:
            sizes = [b - a for a, b in blocks]
            i = int(np.argmax(sizes))
            a, b = blocks[i]
            mid = a + (b - a + 1) // 2
            Rb[mid:b, a:mid] = 0.0
            Rb[a:mid, mid:b] = 0.0
            blocks[i:i + 1] = [(a, mid), (mid, b)]
    return Rb, blocks, normvec


def uniform_pvec(p, b):
    pv = [b] * (p // b)
    if p % b:
        pv.append(p % b)
    return pv


def auto_gamma(R):
    return float(np.linalg.eigvalsh(R)[0])


def r_rr(R, gamma=None):
    g = auto_gamma(R) if gamma is None or gamma < 0 else gamma
    return R + g * np.eye(R.shape[0]), g


def auto_T(R):
    lam = np.linalg.eigvalsh(R)
    lmin = lam[0]
    above = lam[lam > lmin * (1.0 + REL_GAP)]
    return float(above[0])


def r_me(R, T=None):
    """Algorithm 3: R_ME = V diag(max(lambda_k, T)) V^T."""
    lam, V = np.linalg.eigh(R)
    TT = auto_T(R) if T is None or T < 0 else T
    lam_me = np.where(lam <= TT, TT, lam)
    return (V * lam_me) @ V.T, TT


def rhat(R, kind, gamma=None, T=None, block=None):
    """Dense R_hat for kind in {diag, block, rr, me, exact}."""
    if kind == "diag":
        return r_diag(R)
    if kind == "block":
        return r_block(R, uniform_pvec(R.shape[0], block))[0]
    if kind == "rr":
        return r_rr(R, gamma)[0]
    if kind == "me":
        return r_me(R, T)[0]
    if kind == "exact":
        return R.copy()
    raise ValueError(kind)


def dhat(C, ridge=0.0):
    return C + ridge * np.eye(C.shape[0]) if ridge > 0 else C.copy()
