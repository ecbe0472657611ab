"""ctypes binding of the fp64 CPU oracle (oracle/flmisr_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module.  The product path
(paper_2108_04315_b200/) never imports it and shares no code with it.

The C library holds all arithmetic; this module only marshals numpy arrays.
Citations (P:n = PAPER.md line, S:n = SPEC.md line) are in the C source.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "flmisr_oracle.c")
# ORACLE_LIB: an alternative build of this source (tools/mutate_oracle.py points it at mutants)
_LIB = os.environ.get("ORACLE_LIB", os.path.join(_HERE, "libflmisr_oracle.so"))


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no -ffast-math: IEEE fp64 throughout)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Problem(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("lr_h", C.c_int32), ("lr_w", C.c_int32),
        ("shifts", C.POINTER(C.c_double)),
        ("psf", C.POINTER(C.c_double)), ("psf_h", C.c_int32), ("psf_w", C.c_int32),
        ("mag", C.c_int32), ("p_norm", C.c_int32), ("eps", C.c_double),
        ("lam", C.c_double), ("btv_alpha", C.c_double), ("btv_window", C.c_int32),
        ("btv_offsets", C.c_int32),
    ]


class _Stats(C.Structure):
    _fields_ = [("iters_run", C.c_int32), ("accepted", C.c_int32),
                ("converged_at", C.c_int32), ("nonfinite", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        pp = C.POINTER(_Problem)
        _lib.orc_forward.argtypes = [pp, dp, dp]
        _lib.orc_adjoint.argtypes = [pp, dp, dp]
        _lib.orc_value.argtypes = [pp, dp, dp, dp, dp]
        _lib.orc_objective.argtypes = [pp, dp, dp]
        _lib.orc_objective.restype = C.c_double
        _lib.orc_grad.argtypes = [pp, dp, dp, dp]
        _lib.orc_curv.argtypes = [pp, dp, dp, dp]
        _lib.orc_curv.restype = C.c_double
        _lib.orc_init_x0.argtypes = [pp, dp, dp]
        _lib.orc_interp_fuse.argtypes = [pp, dp, dp]
        _lib.orc_scg.argtypes = [pp, dp, dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                 C.c_int, C.c_int, dp, dp, C.POINTER(_Stats), C.c_int]
        _lib.orc_value_rows.argtypes = [pp, dp, dp, C.c_int, C.c_int]
        _lib.orc_value_rows.restype = C.c_double
        _lib.orc_band_bounds.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(C.c_int), C.POINTER(C.c_int)]
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class Problem:
    """The MAP problem of Eq. objective: LR stack geometry, shifts, PSF, SR factor and
    the regularisation weights.  Defaults follow DESIGN.md section 3."""
    k: int
    lr_h: int
    lr_w: int
    shifts: np.ndarray            # k x 2 (dy, dx) LR px
    psf: np.ndarray               # odd x odd, sum 1
    mag: int = 2
    p_norm: int = 1
    eps: float = 1e-3
    lam: float = 0.05
    btv_alpha: float = 0.4
    btv_window: int = 3
    btv_offsets: int = 0          # 0 quadrant, 1 Farsiu (NEXT-4)
    _keep: list = field(default_factory=list, repr=False)

    @property
    def H(self) -> int:
        return self.mag * self.lr_h

    @property
    def W(self) -> int:
        return self.mag * self.lr_w

    def c(self) -> _Problem:
        sh = _f64(self.shifts).reshape(self.k, 2)
        ps = _f64(self.psf)
        self._keep = [sh, ps]
        return _Problem(self.k, self.lr_h, self.lr_w, _dp(sh), _dp(ps), ps.shape[0], ps.shape[1],
                        self.mag, self.p_norm, self.eps, self.lam, self.btv_alpha, self.btv_window,
                        self.btv_offsets)


def forward(pb: Problem, x) -> np.ndarray:
    """y_i = A_i x for every frame (k x lr_h x lr_w)."""
    x = _f64(x).reshape(pb.H, pb.W)
    y = np.zeros((pb.k, pb.lr_h, pb.lr_w))
    c = pb.c()
    assert lib().orc_forward(C.byref(c), _dp(x), _dp(y)) == 0
    return y


def adjoint(pb: Problem, y) -> np.ndarray:
    """sum_i A_i^T y_i (H x W), scatter form."""
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    x = np.zeros((pb.H, pb.W))
    c = pb.c()
    assert lib().orc_adjoint(C.byref(c), _dp(y), _dp(x)) == 0
    return x


def value(pb: Problem, x, y):
    """(D, R): data term and BTV value; J = D + lam * R."""
    x = _f64(x).reshape(pb.H, pb.W)
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    D, R = C.c_double(), C.c_double()
    c = pb.c()
    lib().orc_value(C.byref(c), _dp(x), _dp(y), C.byref(D), C.byref(R))
    return D.value, R.value


def objective(pb: Problem, x, y) -> float:
    x = _f64(x).reshape(pb.H, pb.W)
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    c = pb.c()
    return lib().orc_objective(C.byref(c), _dp(x), _dp(y))


def value_rows(pb: Problem, x, y, lo: int, hi: int) -> float:
    """Band partial f_h over owned rows [lo, hi) (Eq. subfunction)."""
    x = _f64(x).reshape(pb.H, pb.W)
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    c = pb.c()
    return lib().orc_value_rows(C.byref(c), _dp(x), _dp(y), lo, hi)


def grad(pb: Problem, x, y) -> np.ndarray:
    x = _f64(x).reshape(pb.H, pb.W)
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    g = np.zeros((pb.H, pb.W))
    c = pb.c()
    assert lib().orc_grad(C.byref(c), _dp(x), _dp(y), _dp(g)) == 0
    return g


def curv(pb: Problem, x, y, p) -> float:
    """Exact directional curvature p^T Hess J(x) p."""
    x = _f64(x).reshape(pb.H, pb.W)
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    p = _f64(p).reshape(pb.H, pb.W)
    c = pb.c()
    return lib().orc_curv(C.byref(c), _dp(x), _dp(y), _dp(p))


def init_x0(pb: Problem, y) -> np.ndarray:
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    x0 = np.zeros((pb.H, pb.W))
    c = pb.c()
    lib().orc_init_x0(C.byref(c), _dp(y), _dp(x0))
    return x0


def interp_fuse(pb: Problem, y) -> np.ndarray:
    """Multi-image interpolation fusion: LR pixels at their integer HR sites, bilinear elsewhere."""
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    out = np.zeros((pb.H, pb.W))
    c = pb.c()
    lib().orc_interp_fuse(C.byref(c), _dp(y), _dp(out))
    return out


def band_bounds(H: int, g: int, mag: int, h: int):
    lo, hi = C.c_int(), C.c_int()
    lib().orc_band_bounds(H, g, mag, h, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


CURV_EXACT, CURV_FD = 0, 1


RULE_PR_PLUS, RULE_NETLAB = 1, 2


def scg(pb: Problem, y, n_iter: int, x0=None, curv_mode: int = CURV_EXACT, sigma0: float = 1e-4,
        lambda0: float = 1e-6, g: int = 1, eta: int = 2, rules: int = 0):
    """Moller SCG reconstruction (Alg. 1).  Returns (x, trace, stats) where trace is an
    (n_iter+1) x 6 array of (k, f, <r,r>, alpha, lambda_scg, accepted) rows.
    rules: NEXT-4 variants (bit mask RULE_PR_PLUS | RULE_NETLAB; 0 = Moller literal)."""
    y = _f64(y).reshape(pb.k, pb.lr_h, pb.lr_w)
    x = np.zeros((pb.H, pb.W))
    tr = np.zeros((n_iter + 1, 6))
    st = _Stats()
    x0p = None
    if x0 is not None:
        x0a = _f64(x0).reshape(pb.H, pb.W)
        x0p = _dp(x0a)
    c = pb.c()
    rc = lib().orc_scg(C.byref(c), _dp(y), x0p, n_iter, curv_mode, sigma0, lambda0, g, eta,
                       _dp(x), _dp(tr), C.byref(st), rules)
    if rc == -1:
        raise MemoryError("oracle allocation failed")
    stats = dict(iters_run=st.iters_run, accepted=st.accepted, converged_at=st.converged_at,
                 nonfinite=st.nonfinite, rc=rc)
    return x, tr[: st.iters_run + 1], stats
