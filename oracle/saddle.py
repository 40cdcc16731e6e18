"""Saddle operator A and preconditioners P_D, P_I (ORACLE, test infrastructure only).

Definitions:
  A   = [[D, 0, L], [0, R, H], [L^T, H^T, 0]]                       Eq. 2.2
  D   = blkdiag(B, Q_1..Q_N), R = blkdiag(R_0..R_N), H = blkdiag(H_0..H_N)
  P_D = blkdiag(D_hat, R_hat, S_hat),  S_hat = L_hat^T D^{-1} L_hat    Eq. 2.4
  P_I = [[D, 0, L_hat], [0, R_hat, 0], [L_hat^T, 0, 0]]             Eq. 2.4
Matrix-free forms:
  A x    = (D x1 + L x3,  R x2 + H x3,  L^T x1 + H^T x2)
           (P:L638 prints "R x_1"; Eq. 2.2 fixes R x_2 -- reading A22)
  P_D^-1 = (D_hat^-1 x1,  R_hat^-1 x2,  L_hat^-1 D L_hat^-T x3)       P:L651 (exact D, A18)
  P_I^-1 = (c1 = L_hat^-T x3,  R_hat^-1 x2,  L_hat^-1 (x1 - D c1))

Two independent routes:
  * Explicit: assemble the dense matrices above; P^{-1} x is an LU solve with
    the assembled P (np.linalg.solve), never the matrix-free formula.
  * Blockwise: literal per-window loops of P:L629-667 with per-constituent
    counters (R_i, R_hat^-1, D_i, D_hat^-1, M_i), as tabulated in Tables 7.2,
    7.3, S5-S7.
Vectors are in PAPER order for one right-hand side: (eta_0..eta_N, nu_0..nu_N,
x_0..x_N).
"""
from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla

from . import lhat as LH
from . import ichol as IC
from . import rhat as RH
from .models import model_matrices


@dataclass
class Precond:
    shape: str = "PD"      # "PD" | "PI"
    lhat: str = "LM"       # "L0" | "LI" | "LM" | "L"
    k: int = 4
    rhat: str = "exact"    # "diag" | "block" | "rr" | "me" | "exact"
    gamma: float = -1.0
    T: float = -1.0
    block: int = 0
    ridge: float = 0.0
    # Algorithm 1 in full: pvec / tol / maxsize / numproc (None = uniform
    # `block` with every cut applied, reading A7)
    pvec: tuple = None
    block_tol: float = float("inf")
    maxsize: int = 0
    numproc: int = 0
    # "chol": exact Cholesky factors (reading A4); "ichol": IC(0) factors as the paper
    # applies them: the preconditioner block becomes L L^T
    factor: str = "chol"


def selection_matrix(H_idx, s):
    H = np.zeros((len(H_idx), s))
    H[np.arange(len(H_idx)), H_idx] = 1.0
    return H


def csr_matrix(rowptr, col, val, s):
    """Dense H_i from CSR arrays (general observation operator)."""
    p = len(rowptr) - 1
    H = np.zeros((p, s))
    for j in range(p):
        for k in range(rowptr[j], rowptr[j + 1]):
            H[j, col[k]] += val[k]
    return H


def obs_matrix(prob):
    """H_i of a synth.Problem: CSR when given (prob.H_csr), else the selection H_idx."""
    if getattr(prob, "H_csr", None) is not None:
        return csr_matrix(*prob.H_csr, prob.s)
    return selection_matrix(prob.H_idx, prob.s)


class Saddle:
    """One right-hand side's saddle system (M_w may depend on the column)."""

    def __init__(self, prob, col=0, Ms=None):
        self.prob = prob
        self.s, self.p, self.N = prob.s, prob.p, prob.N
        self.W = prob.N + 1
        self.B, self.Q, self.R = prob.B, prob.Q, prob.R
        self.Hi = obs_matrix(prob)
        self.Ms = Ms if Ms is not None else model_matrices(prob, col)
        self.counters = dict(R=0, Rhat_inv=0, D=0, Dhat_inv=0, M=0)
        self._cache = {}

    # ----- helpers ------------------------------------------------------
    def Dblk(self, w):
        return self.B if w == 0 else self.Q

    def split(self, v):
        s, p, W = self.s, self.p, self.W
        x1 = [v[w * s:(w + 1) * s] for w in range(W)]
        o = W * s
        x2 = [v[o + w * p:o + (w + 1) * p] for w in range(W)]
        o += W * p
        x3 = [v[o + w * s:o + (w + 1) * s] for w in range(W)]
        return x1, x2, x3

    @staticmethod
    def join(a, b, c):
        return np.concatenate(list(a) + list(b) + list(c))

    def rhat_matrix(self, pc):
        key = ("Rhat", pc.rhat, pc.gamma, pc.T, pc.block,
               tuple(pc.pvec) if pc.pvec is not None else None, pc.block_tol, pc.maxsize,
               pc.numproc, pc.factor)
        if key not in self._cache:
            if pc.rhat == "block" and pc.pvec is not None:
                M = RH.r_block(self.R, list(pc.pvec), pc.block_tol,
                               pc.maxsize or None, pc.numproc or None)[0]
            else:
                M = RH.rhat(self.R, pc.rhat, pc.gamma, pc.T, pc.block)
            if pc.factor == "ichol" and pc.rhat != "diag":
                assert pc.rhat != "me", "R_ME with IC(0) factors is not supported"
                Lf = IC.ichol0(M)
                M = Lf @ Lf.T
            self._cache[key] = M
        return self._cache[key]

    def dhat_matrix(self, pc, w):
        """D_hat block of window w: D (+ ridge), or L L^T of its IC(0) factor."""
        key = ("Dhat", min(w, 1), pc.ridge, pc.factor)
        if key not in self._cache:
            M = RH.dhat(self.Dblk(w), pc.ridge)
            if pc.factor == "ichol":
                Lf = IC.ichol0(M)
                M = Lf @ Lf.T
            self._cache[key] = M
        return self._cache[key]

    def _spd_solve(self, key, mat_fn, rhs):
        """Solve with an SPD block; the Cholesky factorisation of each distinct
        block is computed once and reused (scipy cho_factor / cho_solve)."""
        if key not in self._cache:
            self._cache[key] = sla.cho_factor(mat_fn())
        return sla.cho_solve(self._cache[key], rhs)

    # ----- explicit assembly ------------------------------------------------
    def assemble_D(self):
        return sla.block_diag(self.B, *([self.Q] * self.N))

    def assemble_A(self):
        s, p, W = self.s, self.p, self.W
        D = self.assemble_D()
        Rb = sla.block_diag(*([self.R] * W))
        H = sla.block_diag(*([self.Hi] * W))
        L = LH.assemble("L", self.Ms, s)
        Z = np.zeros
        return np.block([[D, Z((W * s, W * p)), L],
                         [Z((W * p, W * s)), Rb, H],
                         [L.T, H.T, Z((W * s, W * s))]])

    def assemble_P(self, pc):
        s, p, W = self.s, self.p, self.W
        D = self.assemble_D()
        Rh = sla.block_diag(*([self.rhat_matrix(pc)] * W))
        Lh = LH.assemble(pc.lhat, self.Ms, s, pc.k)
        Z = np.zeros
        if pc.shape == "PD":
            Dh = sla.block_diag(self.dhat_matrix(pc, 0), *([self.dhat_matrix(pc, 1)] * self.N))
            Sh = Lh.T @ np.linalg.solve(D, Lh)
            return sla.block_diag(Dh, Rh, Sh)
        return np.block([[D, Z((W * s, W * p)), Lh],
                         [Z((W * p, W * s)), Rh, Z((W * p, W * s))],
                         [Lh.T, Z((W * s, W * p)), Z((W * s, W * s))]])

    def explicit_apply_A(self, v):
        return self.assemble_A() @ v

    def explicit_apply_Pinv(self, pc, v):
        return np.linalg.solve(self.assemble_P(pc), v)

    # ----- blockwise -------------------------------------------
    def _n_m(self, pc):
        return LH.n_model_blocks(pc.lhat, self.N, pc.k)

    def apply_A(self, v):
        x1, x2, x3 = self.split(v)
        W = self.W
        Lx3 = LH.apply("L", self.Ms, x3)
        LTx1 = LH.apply_T("L", self.Ms, x1)
        c1 = [self.Dblk(w) @ x1[w] + Lx3[w] for w in range(W)]
        c2 = [self.R @ x2[w] + self.Hi @ x3[w] for w in range(W)]
        c3 = [LTx1[w] + self.Hi.T @ x2[w] for w in range(W)]
        c = self.counters
        c["D"] += W
        c["R"] += W
        c["M"] += 2 * self.N
        return self.join(c1, c2, c3)

    def _rhat_inv(self, pc, x2):
        key = ("cho_Rhat", pc.rhat, pc.gamma, pc.T, pc.block,
               tuple(pc.pvec) if pc.pvec is not None else None, pc.block_tol, pc.maxsize,
               pc.numproc, pc.factor)
        self.counters["Rhat_inv"] += self.W
        return [self._spd_solve(key, lambda: self.rhat_matrix(pc), x2[w]) for w in range(self.W)]

    def apply_Pinv(self, pc, v):
        x1, x2, x3 = self.split(v)
        W = self.W
        c = self.counters
        c2 = self._rhat_inv(pc, x2)
        if pc.shape == "PD":
            c1 = [self._spd_solve(("cho_D", min(w, 1), pc.ridge, pc.factor),
                                  lambda w=w: self.dhat_matrix(pc, w), x1[w])
                  for w in range(W)]
            t = LH.solve_T(pc.lhat, self.Ms, x3, pc.k)
            t = [self.Dblk(w) @ t[w] for w in range(W)]
            c3 = LH.solve(pc.lhat, self.Ms, t, pc.k)
            c["Dhat_inv"] += W
        else:
            c1 = LH.solve_T(pc.lhat, self.Ms, x3, pc.k)
            t = [x1[w] - self.Dblk(w) @ c1[w] for w in range(W)]
            c3 = LH.solve(pc.lhat, self.Ms, t, pc.k)
        c["D"] += W
        c["M"] += 2 * self._n_m(pc)
        return self.join(c1, c2, c3)


def primal_solution(sad, b, d):
    """Primal incremental 4D-Var normal equations:
    S dx = L^T D^{-1} b + H^T R^{-1} d with S = L^T D^{-1} L + H^T R^{-1} H;
    then d_eta = D^{-1}(b - L dx), d_nu = R^{-1}(d - H dx).  Dense."""
    s, p, W = sad.s, sad.p, sad.W
    D = sad.assemble_D()
    Rb = sla.block_diag(*([sad.R] * W))
    H = sla.block_diag(*([sad.Hi] * W))
    L = LH.assemble("L", sad.Ms, s)
    Dinv_L = np.linalg.solve(D, L)
    Rinv_H = np.linalg.solve(Rb, H)
    S = L.T @ Dinv_L + H.T @ Rinv_H
    rhs = L.T @ np.linalg.solve(D, b) + H.T @ np.linalg.solve(Rb, d)
    dx = np.linalg.solve(S, rhs)
    deta = np.linalg.solve(D, b - L @ dx)
    dnu = np.linalg.solve(Rb, d - H @ dx)
    return np.concatenate([deta, dnu, dx])
