"""Shared test helpers: run the CPU oracle column by column in library layout."""
import numpy as np

from oracle.models import model_matrices
from oracle.saddle import Precond, Saddle
from synth.layout import from_paper_order, to_paper_order

PC_KEYS = ("shape", "lhat", "k", "rhat", "gamma", "T", "block", "ridge")


def oracle_precond(pc):
    d = dict(pc)
    return Precond(shape=d.get("shape", "PD"), lhat=d.get("lhat", "LM"), k=d.get("k", 4) or 1,
                   rhat=d.get("rhat", "exact"), gamma=d.get("gamma", -1.0), T=d.get("T", -1.0),
                   block=d.get("block", 0), ridge=d.get("ridge", 0.0),
                   pvec=tuple(d["pvec"]) if d.get("pvec") is not None else None,
                   block_tol=d.get("block_tol", float("inf")), maxsize=d.get("maxsize", 0),
                   numproc=d.get("numproc", 0), factor=d.get("factor", "chol"))


class OracleCols:
    """Per-RHS-column oracle saddles (shared M for heat/dense, per column for L96)."""

    def __init__(self, prob, cols=None):
        self.prob = prob
        self.cols = list(range(prob.m)) if cols is None else list(cols)
        shared = None if prob.model == "l96" else model_matrices(prob, 0)
        self.sad = {c: Saddle(prob, col=c, Ms=shared) for c in self.cols}

    def paper(self, vec):
        return to_paper_order(vec, self.prob.s, self.prob.p, self.prob.W, self.prob.m)

    def apply_A(self, vec):
        P = self.paper(vec)
        return {c: self.sad[c].apply_A(P[c]) for c in self.cols}

    def apply_P(self, pc, vec):
        P = self.paper(vec)
        opc = oracle_precond(pc)
        return {c: self.sad[c].apply_Pinv(opc, P[c]) for c in self.cols}


def rel_err_cols(gpu_vec, oracle_dict, prob):
    P = to_paper_order(gpu_vec, prob.s, prob.p, prob.W, prob.m)
    return {c: np.linalg.norm(P[c] - v) / max(np.linalg.norm(v), 1e-300)
            for c, v in oracle_dict.items()}


def seeded_vec(n, seed):
    return np.random.Generator(np.random.PCG64(seed)).standard_normal(n)
