"""Incomplete Cholesky with zero fill (ORACLE, test infrastructure only).

P:L572 / P:L600 / P:L627: the paper applies D_hat^{-1} and R_hat^{-1} "using the
incomplete Cholesky factors computed with the Matlab function ichol with zero-fill,
i.e. using the same sparsity structure as" the matrix.  IC(0) definition: the lower
triangular L with the sparsity pattern P of tril(A) (exact zeros excluded) such that
(L L^T)_ij = A_ij for every (i, j) in P; column by column:
    L_kk = sqrt(A_kk - sum_{j<k} L_kj^2)
    L_ik = (A_ik - sum_{j<k} L_ij L_kj) / L_kk      for i > k, (i, k) in P
(the sums run over the stored entries; fill outside P is dropped).  Dense storage and
plain loops, as the definition reads.  A non-positive pivot raises (Matlab's ichol
errors the same way)."""
import numpy as np


def ichol0(A):
    n = A.shape[0]
    P = np.tril(A != 0.0)
    L = np.zeros_like(A, dtype=np.float64)
    for k in range(n):
        d = A[k, k] - np.dot(L[k, :k], L[k, :k])
        if not d > 0.0:
            raise np.linalg.LinAlgError(f"ichol0: non-positive pivot at {k}")
        L[k, k] = np.sqrt(d)
        for i in range(k + 1, n):
            if P[i, k]:
                L[i, k] = (A[i, k] - np.dot(L[i, :k], L[k, :k])) / L[k, k]
    return L
