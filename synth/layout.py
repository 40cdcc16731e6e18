"""Vector layouts (pure index permutations, no arithmetic of the method).

Library layout (include/wf4dvar.h, "Vector layout"): one contiguous buffer of
n = (2s+p)*W*m doubles holding three segments, each stored [len][W][m]
row-major with the RHS index m fastest:

    delta_eta  [s][W][m]  |  delta_nu  [p][W][m]  |  delta_x  [s][W][m]

Paper layout (Eq. 2.1): per right-hand side, the stacked
vector (delta_eta_0..delta_eta_N, delta_nu_0..delta_nu_N, delta_x_0..delta_x_N),
window-major blocks.  ``to_paper_order`` returns an [m][(2s+p)W] array.
"""
import numpy as np


def pack(eta, nu, x):
    """Concatenate three [len][W][m] segments into the flat library layout."""
    return np.concatenate([np.ascontiguousarray(eta).ravel(),
                           np.ascontiguousarray(nu).ravel(),
                           np.ascontiguousarray(x).ravel()])


def unpack(vec, s, p, W, m):
    """Split a flat library-layout vector into (eta, nu, x) views [len][W][m]."""
    vec = np.asarray(vec)
    n1, n2 = s * W * m, p * W * m
    assert vec.size == 2 * n1 + n2, (vec.size, s, p, W, m)
    eta = vec[:n1].reshape(s, W, m)
    nu = vec[n1:n1 + n2].reshape(p, W, m)
    x = vec[n1 + n2:].reshape(s, W, m)
    return eta, nu, x


def to_paper_order(vec, s, p, W, m):
    """Library layout -> [m][(2s+p)W] paper-ordered vectors (one row per RHS)."""
    eta, nu, x = unpack(vec, s, p, W, m)
    # [len][W][m] -> [m][W][len] -> [m][W*len]
    parts = [np.transpose(a, (2, 1, 0)).reshape(m, -1) for a in (eta, nu, x)]
    return np.concatenate(parts, axis=1)


def from_paper_order(mat, s, p, W):
    """[m][(2s+p)W] paper-ordered vectors -> flat library layout."""
    mat = np.atleast_2d(np.asarray(mat))
    m = mat.shape[0]
    n1, n2 = s * W, p * W
    eta = mat[:, :n1].reshape(m, W, s).transpose(2, 1, 0)
    nu = mat[:, n1:n1 + n2].reshape(m, W, p).transpose(2, 1, 0)
    x = mat[:, n1 + n2:].reshape(m, W, s).transpose(2, 1, 0)
    return pack(eta, nu, x)
