"""Spectral results of the paper as formulas (ORACLE, test infrastructure only).

theorem31_intervals  Theorem 3.1: eigenvalue intervals of P_D^{-1} A.
prop44_unit_count    Prop. 4.4: L_M^{-T} L^T L L_M^{-1} has r*s unit
                     eigenvalues, r = N + 1 - 2 floor(N/k), for 2 <= k <= N+1.
prop45_upper         Prop. 4.5: ||M_i M_i^T|| <= 1  =>  lambda <= k+1+2 sqrt(k).
remark_upper         Remark: lambda <= 1+k+sqrt(k) if k < N <= 2k.
s5_nu                Supp. Prop. S5: non-unit eigenvalues for k = 3,
                     N in {3,4,5}: nu = 1 + (S +- sqrt(S^2 + 4S))/2, S = mu^2+mu^4+mu^6.
s6_upper             Supp. Prop. S6: lambda <= 5 + sqrt(8) for k = 4.
lemma51_map          Lemma 5.1: lambda(R_RR^{-1} R) = lambda/(lambda+gamma).
lemma52_map          Lemma 5.2: lambda(R_ME^{-1} R) = 1 if lambda > T else lambda/T.
"""
import math

import numpy as np


def theorem31_intervals(lamD, LamD, lamR, LamR, lamS, LamS, lamL, LamL, kappaD):
    lp = min(lamD, lamR)
    Lp = max(LamD, LamR)
    neg = ((lp - math.sqrt(lp ** 2 + 4 * Lp * LamS * LamL * kappaD)) / 2,
           (Lp - math.sqrt(Lp ** 2 + 4 * lp * lamS * lamL / kappaD)) / 2)
    mid = (lp, Lp)
    pos = ((lp + math.sqrt(lp ** 2 + 4 * lp * lamS * lamL / kappaD)) / 2,
           (Lp + math.sqrt(Lp ** 2 + 4 * Lp * LamS * LamL * kappaD)) / 2)
    return [neg, mid, pos]


def in_intervals(vals, intervals, rtol=1e-9):
    ok = np.zeros(len(vals), dtype=bool)
    for a, b in intervals:
        pad = rtol * max(1.0, abs(a), abs(b))
        ok |= (vals >= a - pad) & (vals <= b + pad)
    return ok


def prop44_unit_count(N, k, s):
    return (N + 1 - 2 * (N // k)) * s


def prop45_upper(k):
    return k + 1 + 2 * math.sqrt(k)


def remark_upper(k):
    return 1 + k + math.sqrt(k)


def s5_nu(mu):
    S = mu ** 2 + mu ** 4 + mu ** 6
    r = math.sqrt(S * S + 4 * S)
    return 1 + (S - r) / 2, 1 + (S + r) / 2


def s6_upper():
    return 5 + math.sqrt(8)


def lemma51_map(lam, gamma):
    return lam / (lam + gamma)


def lemma52_map(lam, T):
    return np.where(lam > T, 1.0, lam / T)


def gen_eigvals_sym(A, B):
    """Eigenvalues of B^{-1} A for symmetric A and SPD B (dense)."""
    import scipy.linalg as sla
    return sla.eigh(A, B, eigvals_only=True)
