"""Model term L and its approximations (ORACLE, test infrastructure only).

Window indexing: windows w = 0..N (W = N+1); M_w maps window w-1 to w (w=1..N).
The paper's 1-based block (i, j) is window (i-1, j-1).

  L      Eq. 2.3: identity diagonal, -M_w on block (w, w-1).
  L_0    P:L155: the identity.
  L_I    P:L159-168: -I on every sub-diagonal block.
  L_M(k) Def. 4.1: block (j+1, j) (1-based) is -M_j iff j is not
         divisible by k; i.e. 0-based window w keeps -M_w iff w mod k != 0
         (reading A11).  L = L_M(N+1), L_M(1) = I.
  Lemma 4.2: block (i, j) of L_M^{-1} is prod_{m=1}^{i-j} M_{i-m}
         for 1 <= i-j <= (i-1) mod k, identity on the diagonal, 0 otherwise.
"""
import numpy as np


def subdiag_blocks(kind, Ms, k=None):
    """List of the N sub-diagonal blocks (entry for w=1..N is the block that
    multiplies x_{w-1} in row w, WITHOUT the minus sign), or None for zero."""
    N = len(Ms)
    s = Ms[0].shape[0] if N else 0
    out = []
    for w in range(1, N + 1):
        if kind == "L":
            out.append(Ms[w - 1])
        elif kind == "L0":
            out.append(None)
        elif kind == "LI":
            out.append(np.eye(s))
        elif kind == "LM":
            out.append(Ms[w - 1] if (w % k) != 0 else None)
        else:
            raise ValueError(kind)
    return out


def assemble(kind, Ms, s, k=None):
    """Dense (N+1)s x (N+1)s matrix of L / L_0 / L_I / L_M(k)."""
    N = len(Ms)
    W = N + 1
    A = np.eye(W * s)
    for w, blk in enumerate(subdiag_blocks(kind, Ms, k), start=1):
        if blk is not None:
            A[w * s:(w + 1) * s, (w - 1) * s:w * s] = -blk
    return A


def lemma42_inverse(Ms, s, k):
    """L_M(k)^{-1} written out from Lemma 4.2's block formula (1-based i, j)."""
    N = len(Ms)
    W = N + 1
    Minv = np.zeros((W * s, W * s))

    def M(idx):  # paper's M_idx, idx = 1..N
        return Ms[idx - 1]

    for i in range(1, W + 1):
        for j in range(1, W + 1):
            if i == j:
                blk = np.eye(s)
            elif 1 <= i - j <= (i - 1) % k:
                blk = np.eye(s)
                for mm in range(1, i - j + 1):      # prod_{m=1}^{i-j} M_{i-m}
                    blk = blk @ M(i - mm)
            else:
                continue
            Minv[(i - 1) * s:i * s, (j - 1) * s:j * s] = blk
    return Minv


def chains(W, k):
    """Independent index ranges of L_M(k): [c*k, min(c*k+k, W))."""
    return [(c, min(c + k, W)) for c in range(0, W, k)]


def apply(kind, Ms, x, k=None):
    """(L^ x)_w = x_w - B_w x_{w-1}, blocks of x stacked window-major (list)."""
    blocks = subdiag_blocks(kind, Ms, k)
    out = [x[0].copy()]
    for w in range(1, len(x)):
        b = blocks[w - 1]
        out.append(x[w] - (b @ x[w - 1] if b is not None else 0.0))
    return out


def apply_T(kind, Ms, x, k=None):
    """(L^T x)_w = x_w - B_{w+1}^T x_{w+1}."""
    blocks = subdiag_blocks(kind, Ms, k)
    W = len(x)
    out = []
    for w in range(W):
        y = x[w].copy()
        if w + 1 < W and blocks[w] is not None:
            y = y - blocks[w].T @ x[w + 1]
        out.append(y)
    return out


def solve(kind, Ms, r, k=None):
    """L^{-1} r by forward substitution (z_w = r_w + B_w z_{w-1})."""
    blocks = subdiag_blocks(kind, Ms, k)
    z = [r[0].copy()]
    for w in range(1, len(r)):
        b = blocks[w - 1]
        z.append(r[w] + (b @ z[w - 1] if b is not None else 0.0))
    return z


def solve_T(kind, Ms, r, k=None):
    """L^{-T} r by backward substitution (z_w = r_w + B_{w+1}^T z_{w+1})."""
    blocks = subdiag_blocks(kind, Ms, k)
    W = len(r)
    z = [None] * W
    z[W - 1] = r[W - 1].copy()
    for w in range(W - 2, -1, -1):
        b = blocks[w]
        z[w] = r[w] + (b.T @ z[w + 1] if b is not None else 0.0)
    return z


def n_model_blocks(kind, N, k=None):
    """Number of retained M_w blocks (each costs one M and one M^T product per
    L^{-1}/L^{-T} pair): N - floor(N/k) for L_M(k), N for L, 0 for L_0/L_I."""
    if kind == "L":
        return N
    if kind in ("L0", "LI"):
        return 0
    return N - N // k
