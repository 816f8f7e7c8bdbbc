"""ctypes access to the CPU oracle -- TEST INFRASTRUCTURE ONLY.

* liboracle.so     : C restatement of the reference direct solvers (oracle.c).
* _ref/libfractime_ref.so : the unmodified reference library + shim
  (build_ref.sh), when it has been built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module, as the checker.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libfractime_ref.so"

OR_ODE, OR_HYPER, OR_WAVE, OR_DIFFUSION = 0, 1, 2, 3

_o = None
_r = None


def build(reference: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    if reference and Path("/root/reference/proj/src").exists():
        subprocess.run(["bash", str(HERE / "build_ref.sh")], check=True, capture_output=True)


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64).ctypes.data


def olib():
    global _o
    if _o is None:
        if not ORACLE_SO.exists():
            build(reference=False)
        L = C.CDLL(str(ORACLE_SO))
        P, U, D, I = C.c_void_p, C.c_uint64, C.c_double, C.c_int
        L.or_power_step.argtypes = [U, D]
        L.or_power_step.restype = D
        L.or_weights.argtypes = [D, U, P]
        L.or_col_s4.argtypes = [D, U, D, D, P]
        L.or_col_s3.argtypes = [D, U, D, D, P]
        L.or_col_s2.argtypes = [D, U, D, D, P, P]
        L.or_rhs_s2.argtypes = [D, U, U, D, P, P, P]
        L.or_direct_s2.argtypes = [D, U, U, D, D, P, P, P]
        L.or_col_ode.argtypes = [D, U, D, P]
        L.or_rhs_s4.argtypes = [D, U, U, D, P, P, P]
        L.or_rhs_s3.argtypes = [D, U, U, D, P, P, P, I, P]
        L.or_rhs_ode.argtypes = [D, U, D, P, D, P]
        L.or_forward_solve.argtypes = [P, P, U, P]
        L.or_forward_solve.restype = I
        L.or_toeplitz_matvec.argtypes = [P, P, U, P, P]
        L.or_toeplitz_matvec.restype = None
        L.or_block_matvec.argtypes = [P, P, U, U, D, P, P]
        L.or_block_matvec.restype = None
        L.or_direct_s4.argtypes = [D, U, U, D, D, P, P, P]
        L.or_direct_s3.argtypes = [D, U, U, D, D, P, P, P, I, P]
        L.or_march_ld.argtypes = [I, U, U, P, D, P, P]
        L.or_forcing_modes.argtypes = [U, U, D, D, D, D, I, P, P, P, P, P]
        L.or_sine_grid.argtypes = [U, D, D, P]
        L.or_splitmix64.argtypes = [C.POINTER(U)]
        L.or_splitmix64.restype = U
        L.or_uniform.argtypes = [C.POINTER(U)]
        L.or_uniform.restype = D
        L.or_normal.argtypes = [C.POINTER(U)]
        L.or_normal.restype = D
        _o = L
    return _o


def rlib():
    """The unmodified reference (None if it has not been built)."""
    global _r
    if _r is None:
        if not REF_SO.exists():
            return None
        L = C.CDLL(str(REF_SO))
        P, U, D, I = C.c_void_p, C.c_uint64, C.c_double, C.c_int
        L.ref_last_error.restype = C.c_char_p
        L.ref_power_step.argtypes = [U, D]
        L.ref_power_step.restype = D
        L.ref_weights.argtypes = [I, D, U, P]
        L.ref_solve.argtypes = [I, I, D, U, U, D, D, P, P, P, D, U, U, P, C.POINTER(U), C.POINTER(D)]
        L.ref_ode_column.argtypes = [D, U, D, P]
        L.ref_forward_solve.argtypes = [P, P, U, P]
        L.ref_toeplitz_gmres.argtypes = [P, P, U, D, U, P, C.POINTER(U)]
        L.ref_toeplitz_matvec.argtypes = [P, P, U, P, P]
        L.ref_block_matvec.argtypes = [P, P, U, U, D, P, P]
        L.ref_setup.argtypes = [I, D, U, U, D, D, P, P, P, P, P, P]
        _r = L
    return _r


# ---- problem inputs ---------------------------------------------------------

def forcing_grid(w) -> np.ndarray:
    """Sample a workload's separable forcing at the reference's points with glibc
    (x_i = i h, t_n = n tau; wave (n - 1/2) tau; Scheme 2 x = (i - 1/2) h).
    Returns [B*nodes, N]."""
    s0 = w.specs[0]
    N, nodes = s0.time_steps, w.nodes
    ode = int(s0.scheme) == OR_ODE
    shift = -0.5 if int(s0.scheme) == OR_WAVE else 0.0
    xshift = -0.5 if int(s0.scheme) == OR_HYPER else 0.0
    out = np.empty((w.B * nodes, N))
    trig = np.ascontiguousarray(w.trig, dtype=np.int32)
    for b, s in enumerate(w.specs):
        h = 0.0 if ode else s.space_length / s.space_cells
        cells = 2 if ode else s.space_cells
        Fb = np.empty((nodes, N))
        olib().or_forcing_modes(cells, N, h, s.tau(), xshift, shift, len(w.k), _d(w.a[b]), _d(w.k), _d(w.p[b]),
                                trig.ctypes.data, Fb.ctypes.data)
        out[b * nodes:(b + 1) * nodes] = Fb
    return out


def initial_grid(w, amp) -> Optional[np.ndarray]:
    """amp_b * sin(pi x_i) per problem (ODE: amp_b), glibc sin.  Scheme 2 takes
    u0 at x_0 .. x_{cells-1} (its RHS uses u0(x_i) + u0(x_{i-1})): nodes + 1 values
    per problem, the boundary value first."""
    if amp is None:
        return None
    s0 = w.specs[0]
    if int(s0.scheme) == OR_ODE:
        return np.ascontiguousarray(np.asarray(amp, dtype=np.float64))
    if int(s0.scheme) == OR_HYPER:
        out = np.empty(w.B * (w.nodes + 1))
        for b, s in enumerate(w.specs):
            seg = np.empty(w.nodes)
            olib().or_sine_grid(s.space_cells, s.space_length / s.space_cells, float(amp[b]), seg.ctypes.data)
            out[b * (w.nodes + 1)] = float(amp[b]) * 0.0  # amp * sin(pi * 0)
            out[b * (w.nodes + 1) + 1:(b + 1) * (w.nodes + 1)] = seg
        return out
    out = np.empty(w.B * w.nodes)
    for b, s in enumerate(w.specs):
        seg = np.empty(w.nodes)
        olib().or_sine_grid(s.space_cells, s.space_length / s.space_cells, float(amp[b]), seg.ctypes.data)
        out[b * w.nodes:(b + 1) * w.nodes] = seg
    return out


# ---- oracle solvers (fp64 reference order; long double) ----------------------

def direct(w, F, u0=None, phi=None, rhs_mode: int = 0) -> np.ndarray:
    """Reference direct march (restated) for every problem of workload w."""
    s0 = w.specs[0]
    N, nodes = s0.time_steps, w.nodes
    U = np.empty((w.B * nodes, N))
    for b, s in enumerate(w.specs):
        Fb = np.ascontiguousarray(F[b * nodes:(b + 1) * nodes])
        Ub = np.empty((nodes, N))
        u0b = None if (u0 is None or int(s.scheme) == OR_HYPER) else np.ascontiguousarray(u0[b * nodes:(b + 1) * nodes])
        phib = None if phi is None else np.ascontiguousarray(phi[b * nodes:(b + 1) * nodes])
        if int(s.scheme) == OR_HYPER:
            u0h = None if u0 is None else np.ascontiguousarray(u0[b * (nodes + 1):(b + 1) * (nodes + 1)])
            olib().or_direct_s2(s.gamma, s.space_cells, N, s.h(), s.tau(), _d(Fb), _d(u0h), Ub.ctypes.data)
        elif int(s.scheme) == OR_DIFFUSION:
            olib().or_direct_s4(s.gamma, s.space_cells, N, s.h(), s.tau(), _d(Fb), _d(u0b), Ub.ctypes.data)
        elif int(s.scheme) == OR_WAVE:
            olib().or_direct_s3(s.gamma, s.space_cells, N, s.h(), s.tau(), _d(Fb), _d(u0b), _d(phib),
                                rhs_mode, Ub.ctypes.data)
        else:
            col = np.empty(N)
            olib().or_col_ode(s.gamma, N, s.tau(), col.ctypes.data)
            R = np.empty(N)
            olib().or_rhs_ode(s.gamma, N, s.tau(), _d(Fb[0]), float(u0b[0]) if u0b is not None else 0.0,
                              R.ctypes.data)
            olib().or_forward_solve(col.ctypes.data, R.ctypes.data, N, Ub.ctypes.data)
        U[b * nodes:(b + 1) * nodes] = Ub
    return U


def column(s) -> np.ndarray:
    N = s.time_steps
    col = np.empty(N)
    if int(s.scheme) == OR_DIFFUSION:
        olib().or_col_s4(s.gamma, N, s.h(), s.tau(), col.ctypes.data)
    elif int(s.scheme) == OR_HYPER:
        olib().or_col_s2(s.gamma, N, s.h(), s.tau(), col.ctypes.data, None)
    elif int(s.scheme) == OR_WAVE:
        olib().or_col_s3(s.gamma, N, s.h(), s.tau(), col.ctypes.data)
    else:
        olib().or_col_ode(s.gamma, N, s.tau(), col.ctypes.data)
    return col


def march_ld(s, R: np.ndarray) -> np.ndarray:
    """Long-double march of one problem's BLTT system (exact-arithmetic stand-in)."""
    N = s.time_steps
    col = column(s)
    nodes = R.shape[0]
    kind = {OR_ODE: 0, OR_DIFFUSION: 1, OR_WAVE: 2, OR_HYPER: 3}[int(s.scheme)]
    off = 0.0
    if kind == 1:
        off = -1.0 / (s.h() * s.h())
    elif kind == 2:
        off = -1.0 / s.h()
    elif kind == 3:
        b = np.empty(N)
        olib().or_col_s2(s.gamma, N, s.h(), s.tau(), col.ctypes.data, b.ctypes.data)
        off = -float(b[0])
    U = np.empty((nodes, N))
    Rc = np.ascontiguousarray(R, dtype=np.float64)
    olib().or_march_ld(kind, nodes, N, col.ctypes.data, off, Rc.ctypes.data, U.ctypes.data)
    return U


def rhs(w, F, u0=None, phi=None, rhs_mode=0) -> np.ndarray:
    s0 = w.specs[0]
    N, nodes = s0.time_steps, w.nodes
    R = np.empty((w.B * nodes, N))
    for b, s in enumerate(w.specs):
        Fb = np.ascontiguousarray(F[b * nodes:(b + 1) * nodes])
        Rb = np.empty((nodes, N))
        if int(s.scheme) == OR_HYPER:
            u0h = None if u0 is None else np.ascontiguousarray(u0[b * (nodes + 1):(b + 1) * (nodes + 1)])
            olib().or_rhs_s2(s.gamma, s.space_cells, N, s.tau(), _d(Fb), _d(u0h), Rb.ctypes.data)
        elif int(s.scheme) == OR_DIFFUSION:
            u0b = None if u0 is None else np.ascontiguousarray(u0[b * nodes:(b + 1) * nodes])
            olib().or_rhs_s4(s.gamma, s.space_cells, N, s.tau(), _d(Fb), _d(u0b), Rb.ctypes.data)
        elif int(s.scheme) == OR_WAVE:
            u0b = None if u0 is None else np.ascontiguousarray(u0[b * nodes:(b + 1) * nodes])
            phib = None if phi is None else np.ascontiguousarray(phi[b * nodes:(b + 1) * nodes])
            olib().or_rhs_s3(s.gamma, s.space_cells, N, s.tau(), _d(Fb), _d(u0b), _d(phib), rhs_mode,
                             Rb.ctypes.data)
        else:
            olib().or_rhs_ode(s.gamma, N, s.tau(), _d(Fb[0]), float(u0[b]) if u0 is not None else 0.0,
                              Rb.ctypes.data)
        R[b * nodes:(b + 1) * nodes] = Rb
    return R


def ref_solve(s, method: str, F, u0=None, phi=None, tol=0.0, restart=0, max_iter=0):
    """Run the UNMODIFIED reference solve() on the same inputs."""
    L = rlib()
    if L is None:
        raise RuntimeError("reference library not built (oracle/build_ref.sh)")
    nodes = s.space_cells - 1
    U = np.empty((nodes, s.time_steps))
    it = C.c_uint64(0)
    sec = C.c_double(0.0)
    rc = L.ref_solve(int(s.scheme), 2 if method == "direct" else 3, s.gamma, s.time_steps, s.space_cells,
                     s.time_length, s.space_length, _d(F), _d(u0), _d(phi), tol, restart, max_iter,
                     U.ctypes.data, C.byref(it), C.byref(sec))
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return U, int(it.value), float(sec.value)


def ref_setup(s, F=None, u0=None):
    """The reference's own scheme assembly: (first column, second column (Scheme 2
    B~) or None, off-block scale (Scheme 4) or None, assembled RHS (Scheme 4, when
    F is given) or None)."""
    L = rlib()
    if L is None:
        raise RuntimeError("reference library not built (oracle/build_ref.sh)")
    N = s.time_steps
    col = np.empty(N)
    col2 = np.empty(N) if int(s.scheme) == OR_HYPER else None
    off = C.c_double(0.0)
    R = np.empty((s.space_cells - 1, N)) if (F is not None and int(s.scheme) == OR_DIFFUSION) else None
    rc = L.ref_setup(int(s.scheme), s.gamma, N, s.space_cells, s.time_length, s.space_length, _d(F), _d(u0),
                     col.ctypes.data, None if col2 is None else col2.ctypes.data, C.byref(off),
                     None if R is None else R.ctypes.data)
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return col, col2, (off.value if int(s.scheme) == OR_DIFFUSION else None), R


def toeplitz_case(n: int, seed: int, lower: bool = False):
    """Seeded Toeplitz test operator (first column, first row), decaying off the
    diagonal, diagonal 4 (well conditioned for the lower-triangular solves)."""
    rng = np.random.default_rng(seed)
    col = rng.standard_normal(n) / (1.0 + np.arange(n)) ** 0.7
    row = rng.standard_normal(n) / (1.0 + np.arange(n)) ** 0.7
    col[0] = 4.0
    row[0] = col[0]
    if lower:
        row[1:] = 0.0
    return col, row


def relerr(x, y) -> float:
    """Normwise  max|x - y| / max|y|."""
    x = np.asarray(x)
    y = np.asarray(y)
    return float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300))
