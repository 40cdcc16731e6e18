"""ctypes binding of libwf4dvar.so (include/wf4dvar.h): argument marshalling only.

Every step of the hot path runs in the CUDA library; this module converts
Python/NumPy/torch arguments into the C structs and pointers of the ABI.
There is no fallback: if the shared library is missing or fails to load,
importing this module raises.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libwf4dvar.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build it with `python -m paper_2105_06975_b200.build` "
        "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- structs
M_DENSE, M_HEAT, M_L96, M_HEAT_EXPLICIT = 0, 1, 2, 3
PD, PI = 0, 1
L0, LI, LM, LEXACT = 0, 1, 2, 3
RDIAG, RBLOCK, RRR, RME, REXACT = 0, 1, 2, 3, 4
MINRES, GMRES = 0, 1
STATUS = {0: "OK", 1: "EINVAL", 2: "ENOTSPD", 3: "EINDEF", 4: "ENOCONV", 5: "ECUDA",
          6: "ENCCL", 7: "ENOMEM"}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class Problem(C.Structure):
    _fields_ = [("s", C.c_int32), ("p", C.c_int32), ("N", C.c_int32), ("m", C.c_int32),
                ("B", _dp), ("Q", _dp), ("R", _dp), ("H_idx", _ip), ("model", C.c_int32),
                ("M_dense", _dp), ("heat_r", C.c_double), ("l96_traj", _dp),
                ("l96_F", C.c_double), ("l96_dt", C.c_double), ("l96_nsub", C.c_int32),
                ("heat_nsteps", C.c_int32), ("H_rowptr", _ip), ("H_col", _ip), ("H_val", _dp)]


class Precond(C.Structure):
    _fields_ = [("shape", C.c_int32), ("lhat", C.c_int32), ("k", C.c_int32), ("rhat", C.c_int32),
                ("gamma", C.c_double), ("T", C.c_double), ("block", C.c_int32),
                ("dhat_ridge", C.c_double), ("pvec", _ip), ("npvec", C.c_int32),
                ("block_tol", C.c_double), ("maxsize", C.c_int32), ("numproc", C.c_int32),
                ("factor", C.c_int32), ("apply_mode", C.c_int32)]


TRANSPORT_NONE, TRANSPORT_NCCL, TRANSPORT_LOCAL = 0, 1, 2


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32),
                ("stream", C.c_void_p), ("transport", C.c_int32), ("nccl_id", C.c_void_p),
                ("local_group", C.c_void_p)]


class ChainStep(C.Structure):
    _fields_ = [("j", C.c_int32), ("recv", C.c_int32), ("send", C.c_int32), ("nl", C.c_int32),
                ("first", C.c_int32 * 2), ("stride", C.c_int32 * 2), ("count", C.c_int32 * 2)]


class SolveOpts(C.Structure):
    _fields_ = [("solver", C.c_int32), ("tol", C.c_double), ("maxit", C.c_int32),
                ("restart", C.c_int32), ("mark_tol", C.c_double), ("check_every", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iters", _ip), ("relres", _dp), ("converged", C.POINTER(C.c_uint8)),
                ("history", _dp), ("seconds", C.c_double), ("seconds_to_mark", C.c_double),
                ("iters_to_mark", C.c_int32), ("n_apply_A", C.c_int64), ("n_apply_P", C.c_int64),
                ("n_R", C.c_int64), ("n_Rhat_inv", C.c_int64), ("n_D", C.c_int64),
                ("n_Dhat_inv", C.c_int64), ("n_M", C.c_int64), ("seconds_init", C.c_double)]


class KStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


_ctx = C.c_void_p
_sig = {
    "wf4dvar_create": (C.c_int, [C.POINTER(Problem), C.POINTER(Precond), C.POINTER(Dist), C.POINTER(_ctx)]),
    "wf4dvar_set_precond": (C.c_int, [_ctx, C.POINTER(Precond)]),
    "wf4dvar_destroy": (C.c_int, [_ctx]),
    "wf4dvar_local_windows": (C.c_int, [_ctx, _ip, _ip]),
    "wf4dvar_vector_len": (C.c_int, [_ctx, C.POINTER(C.c_int64)]),
    "wf4dvar_apply_A": (C.c_int, [_ctx, C.c_void_p, C.c_void_p]),
    "wf4dvar_apply_P": (C.c_int, [_ctx, C.c_void_p, C.c_void_p]),
    "wf4dvar_apply_AP": (C.c_int, [_ctx, C.c_void_p, C.c_void_p, C.c_void_p]),
    "wf4dvar_apply_AP_host": (C.c_int, [_ctx, C.c_void_p, C.c_void_p]),
    "wf4dvar_solve": (C.c_int, [_ctx, C.c_void_p, C.c_void_p, C.POINTER(SolveOpts), C.POINTER(Report)]),
    "wf4dvar_solve_host": (C.c_int, [_ctx, C.c_void_p, C.c_void_p, C.POINTER(SolveOpts), C.POINTER(Report)]),
    "wf4dvar_outer_loop": (C.c_int, [_ctx, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                     C.POINTER(SolveOpts), _ip, _dp, _dp]),
    "wf4dvar_lanczos": (C.c_int, [_ctx, C.c_int32, C.c_void_p, C.c_int32, _dp, _dp, _dp, _dp]),
    "wf4dvar_profile_enable": (C.c_int, [_ctx, C.c_int32]),
    "wf4dvar_profile_read": (C.c_int, [_ctx, C.POINTER(KStat), C.c_int32, _ip]),
    "wf4dvar_launch_count": (C.c_int64, [_ctx]),
    "wf4dvar_partition": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, _ip, _ip]),
    "wf4dvar_chain_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(ChainStep), C.c_int32, _ip]),
    "wf4dvar_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "wf4dvar_rblock_plan": (C.c_int, [_dp, C.c_int32, _ip, C.c_int32, C.c_double, C.c_int32,
                                      C.c_int32, _ip, C.c_int32, _ip]),
    "wf4dvar_local_group_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "wf4dvar_local_group_destroy": (C.c_int, [C.c_void_p]),
    "wf4dvar_last_error": (C.c_char_p, [_ctx]),
    "wf4dvar_version": (C.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig.keys())


class WF4DVarError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.code = STATUS.get(status, str(status))


def version():
    return _lib.wf4dvar_version().decode()


def partition(W, world, rank):
    """Global windows [w_begin, w_end) owned by `rank` (host only)."""
    b, e = C.c_int32(), C.c_int32()
    st = _lib.wf4dvar_partition(int(W), int(world), int(rank), C.byref(b), C.byref(e))
    if st != 0:
        raise WF4DVarError(st, f"partition(W={W}, world={world}, rank={rank})")
    return b.value, e.value


def chain_plan(W, k, w_begin, w_end, transpose):
    """The library's L_hat chain schedule for the local windows (host only)."""
    n = C.c_int32()
    st = _lib.wf4dvar_chain_plan(int(W), int(k), int(w_begin), int(w_end), int(transpose),
                                 None, 0, C.byref(n))
    if st != 0:
        raise WF4DVarError(st, "chain_plan")
    arr = (ChainStep * max(n.value, 1))()
    _lib.wf4dvar_chain_plan(int(W), int(k), int(w_begin), int(w_end), int(transpose), arr,
                            n.value, C.byref(n))
    return [dict(j=a.j, recv=a.recv, send=a.send,
                 launches=[(a.first[l], a.stride[l], a.count[l]) for l in range(a.nl)])
            for a in arr[:n.value]]


def rblock_plan(R, pvec, block_tol=float("inf"), maxsize=0, numproc=0):
    """Algorithm 1 block boundaries the library computes for R_block (host only):
    list of (start, end) diagonal blocks."""
    R = np.ascontiguousarray(R, dtype=np.float64)
    pv = np.ascontiguousarray(pvec, dtype=np.int32)
    out = np.zeros(pv.size + 3, np.int32)
    n = C.c_int32()
    st = _lib.wf4dvar_rblock_plan(_np_ptr(R, C.c_double), int(R.shape[0]), _np_ptr(pv, C.c_int32),
                                  int(pv.size), float(block_tol), int(maxsize), int(numproc),
                                  _np_ptr(out, C.c_int32), int(out.size), C.byref(n))
    if st != 0:
        raise WF4DVarError(st, _lib.wf4dvar_last_error(None).decode())
    e = out[:n.value].tolist()
    return list(zip(e[:-1], e[1:]))


def nccl_unique_id():
    """128-byte ncclUniqueId (rank 0 creates it; the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    st = _lib.wf4dvar_nccl_unique_id(buf)
    if st != 0:
        raise WF4DVarError(st, _lib.wf4dvar_last_error(None).decode())
    return buf.raw


class LocalGroup:
    """In-process transport group: `world` contexts driven by `world` host threads."""

    def __init__(self, world):
        self._h = C.c_void_p()
        st = _lib.wf4dvar_local_group_create(int(world), C.byref(self._h))
        if st != 0:
            raise WF4DVarError(st, "local_group_create")
        self.world = int(world)

    def close(self):
        if self._h:
            _lib.wf4dvar_local_group_destroy(self._h)
            self._h = None


def local_windows(vec, s, p, W, m, w_begin, w_end):
    """Rank-local part [(2s+p)][w_begin:w_end][m] of a global library-layout vector
    (argument marshalling for the sharded path; numpy or torch)."""
    segs, off = [], 0
    for ln in (s, p, s):
        seg = vec[off:off + ln * W * m].reshape(ln, W, m)[:, w_begin:w_end, :]
        segs.append(seg.reshape(-1))
        off += ln * W * m
    if hasattr(vec, "data_ptr"):
        import torch
        return torch.cat(segs).contiguous()
    return np.ascontiguousarray(np.concatenate(segs))


def global_windows(parts, s, p, m, bounds):
    """Inverse of local_windows: assemble rank-local vectors (in rank order, with
    their (w_begin, w_end)) into one global library-layout numpy vector."""
    W = bounds[-1][1]
    out = []
    for si, ln in enumerate((s, p, s)):
        blocks = []
        for v, (b, e) in zip(parts, bounds):
            v = np.asarray(v)
            lw = e - b
            offs = [0, s * lw * m, (s + p) * lw * m]
            blocks.append(v[offs[si]:offs[si] + ln * lw * m].reshape(ln, lw, m))
        out.append(np.concatenate(blocks, axis=1).reshape(-1))
    return np.concatenate(out)


def _ptr(a):
    """Device/host pointer of a torch tensor or numpy array (float64, contiguous)."""
    if hasattr(a, "data_ptr"):
        import torch
        assert a.dtype == torch.float64 and a.is_contiguous(), "need contiguous float64"
        return C.c_void_p(a.data_ptr())
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "need contiguous float64"
    return C.c_void_p(a.ctypes.data)


def _np_ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


SHAPES = {"PD": PD, "PI": PI}
LHATS = {"L0": L0, "LI": LI, "LM": LM, "L": LEXACT}
RHATS = {"diag": RDIAG, "block": RBLOCK, "rr": RRR, "me": RME, "exact": REXACT}


def make_precond(shape="PD", lhat="LM", k=4, rhat="exact", gamma=-1.0, T=-1.0, block=0,
                 ridge=0.0, pvec=None, block_tol=float("inf"), maxsize=0, numproc=0,
                 factor="chol", apply_mode="trsm"):
    pc = Precond(SHAPES[shape], LHATS[lhat], int(k or 1), RHATS[rhat], float(gamma), float(T),
                 int(block or 0), float(ridge))
    if pvec is not None:
        arr = np.ascontiguousarray(pvec, dtype=np.int32)
        pc._pvec_keep = arr            # the library copies it during create/set_precond
        pc.pvec = _np_ptr(arr, C.c_int32)
        pc.npvec = int(arr.size)
    pc.block_tol = float(block_tol)
    pc.maxsize = int(maxsize or 0)
    pc.numproc = int(numproc or 0)
    pc.factor = {"chol": 0, "ichol": 1}[factor]
    pc.apply_mode = {"trsm": 0, "inverse": 1}[apply_mode]
    return pc


class Context:
    """One wf4dvar context on one CUDA device (see include/wf4dvar.h)."""

    def __init__(self, s, p, N, m, B, Q, R, H_idx, model="heat", heat_r=0.25, M_dense=None,
                 l96_traj=None, l96_F=8.0, l96_dt=0.025, l96_nsub=5, precond=None, device=0,
                 stream=None, rank=0, world=1, nccl_id=None, local_group=None, heat_nsteps=1,
                 H_csr=None):
        keep = []

        def arr(a, dt=np.float64):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a

        Bh, Qh, Rh = arr(B), arr(Q), arr(R)
        Hh = arr(H_idx, np.int32)
        pr = Problem()
        pr.s, pr.p, pr.N, pr.m = int(s), int(p), int(N), int(m)
        pr.B, pr.Q, pr.R = _np_ptr(Bh, C.c_double), _np_ptr(Qh, C.c_double), _np_ptr(Rh, C.c_double)
        if Hh is not None:
            pr.H_idx = _np_ptr(Hh, C.c_int32)
        if H_csr is not None:
            rp, cl, vl = arr(H_csr[0], np.int32), arr(H_csr[1], np.int32), arr(H_csr[2])
            pr.H_rowptr, pr.H_col, pr.H_val = (_np_ptr(rp, C.c_int32), _np_ptr(cl, C.c_int32),
                                               _np_ptr(vl, C.c_double))
        pr.heat_nsteps = int(heat_nsteps)
        pr.model = {"dense": M_DENSE, "heat": M_HEAT, "l96": M_L96,
                    "heat_explicit": M_HEAT_EXPLICIT}[model]
        pr.heat_r = float(heat_r)
        if M_dense is not None:
            pr.M_dense = _np_ptr(arr(M_dense), C.c_double)
        if l96_traj is not None:
            pr.l96_traj = _np_ptr(arr(l96_traj), C.c_double)
        pr.l96_F, pr.l96_dt, pr.l96_nsub = float(l96_F), float(l96_dt), int(l96_nsub)
        pc = precond if isinstance(precond, Precond) else make_precond(**(precond or {}))
        transport = TRANSPORT_NONE
        idbuf = None
        if world > 1 or nccl_id is not None or local_group is not None:
            if local_group is not None:
                transport = TRANSPORT_LOCAL
            else:
                assert nccl_id is not None and len(nccl_id) == 128, "world > 1 needs nccl_id"
                transport = TRANSPORT_NCCL
                idbuf = C.create_string_buffer(bytes(nccl_id), 128)
                keep.append(idbuf)
        d = Dist(int(rank), int(world), int(device), C.c_void_p(stream) if stream else None,
                 transport, C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                 local_group._h if local_group is not None else None)
        h = _ctx()
        st = _lib.wf4dvar_create(C.byref(pr), C.byref(pc), C.byref(d), C.byref(h))
        if st != 0:
            raise WF4DVarError(st, _lib.wf4dvar_last_error(None).decode())
        self._h = h
        self.s, self.p, self.N, self.m = int(s), int(p), int(N), int(m)
        self.W = self.N + 1
        self.rank, self.world = int(rank), int(world)
        b, e = C.c_int32(), C.c_int32()
        self._check(_lib.wf4dvar_local_windows(h, C.byref(b), C.byref(e)))
        self.w_begin, self.w_end = b.value, e.value
        n = C.c_int64()
        self._check(_lib.wf4dvar_vector_len(h, C.byref(n)))
        self.n = n.value

    @classmethod
    def from_problem(cls, prob, precond=None, **kw):
        return cls(prob.s, prob.p, prob.N, prob.m, prob.B, prob.Q, prob.R, prob.H_idx,
                   model=prob.model, heat_r=getattr(prob, "heat_r", 0.25),
                   M_dense=getattr(prob, "M_dense", None), l96_traj=getattr(prob, "traj", None),
                   l96_F=getattr(prob, "F", 8.0), l96_dt=getattr(prob, "dt", 0.025),
                   l96_nsub=getattr(prob, "nsub", 5), precond=precond,
                   heat_nsteps=getattr(prob, "heat_nsteps", 1),
                   H_csr=getattr(prob, "H_csr", None), **kw)

    def _check(self, st):
        if st != 0:
            raise WF4DVarError(st, _lib.wf4dvar_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            _lib.wf4dvar_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_precond(self, **kw):
        pc = make_precond(**kw)
        self._check(_lib.wf4dvar_set_precond(self._h, C.byref(pc)))

    def apply_A(self, x, y):
        self._check(_lib.wf4dvar_apply_A(self._h, _ptr(x), _ptr(y)))

    def apply_P(self, x, y):
        self._check(_lib.wf4dvar_apply_P(self._h, _ptr(x), _ptr(y)))

    def apply_AP(self, x, t, y):
        self._check(_lib.wf4dvar_apply_AP(self._h, _ptr(x), _ptr(t), _ptr(y)))

    def apply_AP_host(self, x_host, y_host):
        self._check(_lib.wf4dvar_apply_AP_host(self._h, _ptr(x_host), _ptr(y_host)))

    def _solve(self, fn, rhs, x, solver, tol, maxit, restart, mark_tol, check_every, history):
        opts = SolveOpts({"minres": MINRES, "gmres": GMRES}[solver], float(tol), int(maxit),
                         int(restart), float(mark_tol), int(check_every))
        its = np.zeros(self.m, np.int32)
        rel = np.zeros(self.m, np.float64)
        conv = np.zeros(self.m, np.uint8)
        hist = np.zeros((maxit + 1) * self.m, np.float64) if history else None
        rep = Report()
        rep.iters, rep.relres = _np_ptr(its, C.c_int32), _np_ptr(rel, C.c_double)
        rep.converged = _np_ptr(conv, C.c_uint8)
        if hist is not None:
            rep.history = _np_ptr(hist, C.c_double)
        st = fn(self._h, _ptr(rhs), _ptr(x), C.byref(opts), C.byref(rep))
        if st not in (0, 4):
            self._check(st)
        out = dict(status=STATUS[st], iters=its, relres=rel, converged=conv.astype(bool),
                   seconds=rep.seconds, seconds_to_mark=rep.seconds_to_mark,
                   iters_to_mark=rep.iters_to_mark, n_apply_A=rep.n_apply_A,
                   n_apply_P=rep.n_apply_P, n_R=rep.n_R, n_Rhat_inv=rep.n_Rhat_inv, n_D=rep.n_D,
                   n_Dhat_inv=rep.n_Dhat_inv, n_M=rep.n_M, seconds_init=rep.seconds_init)
        if hist is not None:
            out["history"] = hist.reshape(maxit + 1, self.m)
        return out

    def solve(self, rhs, x, solver="gmres", tol=1e-10, maxit=1000, restart=50, mark_tol=1e-8,
              check_every=1, history=False):
        return self._solve(_lib.wf4dvar_solve, rhs, x, solver, tol, maxit, restart, mark_tol,
                           check_every, history)

    def solve_host(self, rhs, x, solver="gmres", tol=1e-10, maxit=1000, restart=50,
                   mark_tol=1e-8, check_every=1, history=False):
        return self._solve(_lib.wf4dvar_solve_host, rhs, x, solver, tol, maxit, restart,
                           mark_tol, check_every, history)

    def outer_loop(self, xb, y, x, n_outer, solver="gmres", tol=1e-10, maxit=1000, restart=50,
                   check_every=1):
        """Gauss-Newton outer loops (device xb [s][m], y [p][W][m], x [s][W][m] in/out)."""
        opts = SolveOpts({"minres": MINRES, "gmres": GMRES}[solver], float(tol), int(maxit),
                         int(restart), float(tol), int(check_every))
        its = np.zeros(n_outer * self.m, np.int32)
        dxn = np.zeros(n_outer * self.m)
        res = np.zeros(n_outer * self.m)
        self._check(_lib.wf4dvar_outer_loop(self._h, _ptr(xb) if xb is not None else None,
                                            _ptr(y), _ptr(x), int(n_outer), C.byref(opts),
                                            _np_ptr(its, C.c_int32), _np_ptr(dxn, C.c_double),
                                            _np_ptr(res, C.c_double)))
        return dict(inner_iters=its.reshape(n_outer, self.m),
                    dx_norm=np.sqrt(dxn.reshape(n_outer, self.m)),
                    res_norm=np.sqrt(res.reshape(n_outer, self.m)))

    def lanczos(self, op, v0, steps, tridiag=False):
        """Extreme Ritz values per RHS of P_D^{-1} A (op="PA") or L_hat^{-T} L^T L L_hat^{-1}
        (op="LHAT") after `steps` batched Lanczos steps from the device vector v0."""
        lo = np.zeros(self.m)
        hi = np.zeros(self.m)
        a = np.zeros(steps * self.m) if tridiag else None
        b = np.zeros(steps * self.m) if tridiag else None
        self._check(_lib.wf4dvar_lanczos(self._h, {"PA": 0, "LHAT": 1}[op], _ptr(v0), int(steps),
                                         _np_ptr(lo, C.c_double), _np_ptr(hi, C.c_double),
                                         _np_ptr(a, C.c_double) if tridiag else None,
                                         _np_ptr(b, C.c_double) if tridiag else None))
        if tridiag:
            return lo, hi, a.reshape(steps, self.m), b.reshape(steps, self.m)
        return lo, hi

    def profile_enable(self, on=True):
        self._check(_lib.wf4dvar_profile_enable(self._h, 1 if on else 0))

    def profile_read(self):
        arr = (KStat * 32)()
        n = C.c_int32()
        self._check(_lib.wf4dvar_profile_read(self._h, arr, 32, C.byref(n)))
        return {arr[i].name.decode(): dict(launches=arr[i].launches, ms=arr[i].ms,
                                           flops=arr[i].flops, bytes=arr[i].bytes)
                for i in range(n.value)}

    @property
    def launch_count(self):
        return int(_lib.wf4dvar_launch_count(self._h))


# ------------------------------------------------ kernel test hooks (wf4dvar_testing.h)
_lib.wf4dvar_test_gemm.restype = C.c_int
_lib.wf4dvar_test_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_int64,
                                   C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64,
                                   C.c_void_p, C.c_int64, C.c_void_p]
_lib.wf4dvar_test_trsm.restype = C.c_int
_lib.wf4dvar_test_trsm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
TEST_EXPORTED = ("wf4dvar_test_gemm", "wf4dvar_test_trsm")


def test_gemm(A, X, Y, alpha=1.0, beta=0.0, Z=None, stream=None):
    """Y = alpha A X + beta Z on torch float64 CUDA matrices (row-major, may be strided views)."""
    M, K = A.shape
    N = X.shape[1]
    st = _lib.wf4dvar_test_gemm(M, N, K, alpha, C.c_void_p(A.data_ptr()), A.stride(0),
                                C.c_void_p(X.data_ptr()), X.stride(0), beta,
                                C.c_void_p(Z.data_ptr()) if Z is not None else None,
                                Z.stride(0) if Z is not None else 0,
                                C.c_void_p(Y.data_ptr()), Y.stride(0),
                                C.c_void_p(stream) if stream else None)
    if st:
        raise WF4DVarError(st, "wf4dvar_test_gemm")


def test_trsm(G, X, Y, upper=False, blk=0, stream=None):
    """Y = G^{-1} X (lower) or U^{-1} X (upper) for contiguous torch float64 CUDA tensors."""
    n, ncols = X.shape
    assert G.is_contiguous() and X.is_contiguous() and Y.is_contiguous(), "row-major contiguous"
    st = _lib.wf4dvar_test_trsm(n, ncols, 1 if upper else 0, blk, C.c_void_p(G.data_ptr()),
                                C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()),
                                C.c_void_p(stream) if stream else None)
    if st:
        raise WF4DVarError(st, "wf4dvar_test_trsm")
