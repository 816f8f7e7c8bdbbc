"""fractime-b200: B200-native fast solver for the L1-Caputo BLTT systems.

Python host mirror of the reference's solver interface (reference
include/fractime/schemes.hpp): ``ProblemSpec``, ``SchemeId``, ``SolveMethod``,
``solve(spec, method)`` returning a ``SchemeSolution`` with a ``SolutionGrid``
and a ``SolveReport``.  Everything is a thin ctypes layer over the C ABI of
``libfractime_b200.so`` (include/fractime_b200.h); all arithmetic runs in the
CUDA kernels of that library.  There is no CPU path: if the library or a CUDA
device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libfractime_b200.so"
if __import__("os").environ.get("FT_LIB_VARIANT"):  # A/B builds (scratch experiments): an alternative .so
    LIB_PATH = Path(__import__("os").environ["FT_LIB_VARIANT"])


class FractimeError(RuntimeError):
    """Raised for FT_E* codes; .code holds the C ABI code."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(FractimeError, ValueError):
    pass


class DomainError(FractimeError, ValueError):
    pass


class SchemeId(enum.IntEnum):  # reference schemes.hpp:182
    Ode = 0
    Hyperbolic = 1      # Scheme 2 (transport, 0 < gamma < 1)
    DiffusionWave = 2
    Diffusion = 3


class SolveMethod(enum.Enum):  # reference schemes.hpp:184 (Dense/Cg are Scheme 1 only)
    Direct = "direct"
    Fast = "fast"


FT_RHS_REFERENCE = 0
FT_RHS_CORRECTED_N1 = 1


class _Problem(C.Structure):
    _fields_ = [("scheme", C.c_int), ("gamma", C.c_double), ("time_steps", C.c_uint64),
                ("space_cells", C.c_uint64), ("time_length", C.c_double),
                ("space_length", C.c_double)]


class _Options(C.Structure):
    _fields_ = [("rhs_mode", C.c_int), ("near_field", C.c_int), ("device", C.c_int),
                ("flags", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("method", C.c_char * 16), ("iterations", C.c_uint64), ("residual", C.c_double),
                ("seconds", C.c_double), ("device_ms", C.c_double),
                ("kernel_launches", C.c_uint64)]


class _OpTime(C.Structure):
    _fields_ = [("kind", C.c_int), ("level", C.c_int), ("t0", C.c_uint64), ("len", C.c_uint64),
                ("bytes", C.c_uint64), ("ms", C.c_float)]


class _Info(C.Structure):
    _fields_ = [("problems", C.c_uint64), ("nodes", C.c_uint64), ("time_steps", C.c_uint64),
                ("leaf", C.c_uint64), ("levels", C.c_uint64), ("slabs", C.c_uint64),
                ("h", C.c_double), ("tau", C.c_double), ("mu", C.c_double), ("c", C.c_double),
                ("rank", C.c_int), ("world", C.c_int), ("node_begin", C.c_uint64), ("local_nodes", C.c_uint64),
                ("slabs_local", C.c_uint64), ("flags", C.c_uint64)]


PLAN_SLAB_LEAF, PLAN_FUSED_LEAF, PLAN_FUSE0, PLAN_CLUSTER_MP, PLAN_SPLIT_MP, PLAN_ODE_WHOLE = 1, 2, 4, 8, 16, 32


FORCING_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_double, C.c_void_p)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_void_p)
INITIAL_FN = C.CFUNCTYPE(C.c_double, C.c_double, C.c_void_p)

_lib = None

ABI_SYMBOLS = ("ft_setup", "ft_setup_batch", "ft_setup_partitioned", "ft_set_exchange", "ft_plan_get_info", "ft_column", "ft_assemble_rhs",
               "ft_assemble_rhs_grid", "ft_assemble_rhs_modes", "ft_solve_fast", "ft_solve_direct",
               "ft_solve_fast_modes", "ft_p2p_handle", "ft_p2p_connect",
               "ft_profile_fast", "ft_schedule", "ft_set_stream", "ft_last_error", "ft_destroy",
               "ft_setup_toeplitz", "ft_toeplitz_matvec", "ft_block_matvec", "ft_apply", "ft_residual", "ft_nccl_unique_id", "ft_nccl_init")


def lib() -> C.CDLL:
    """Load libfractime_b200.so (build it with __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FractimeError(-5, f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        P, D, U64, I = C.c_void_p, C.POINTER(C.c_double), C.c_uint64, C.c_int
        L.ft_setup.argtypes = [C.POINTER(_Problem), C.POINTER(_Options), C.POINTER(P)]
        L.ft_setup_batch.argtypes = [C.POINTER(_Problem), U64, C.POINTER(_Options), C.POINTER(P)]
        L.ft_setup_partitioned.argtypes = [C.POINTER(_Problem), C.POINTER(_Options), I, I, C.POINTER(P)]
        L.ft_setup_toeplitz.argtypes = [P, U64, U64, C.POINTER(_Options), C.POINTER(P)]
        L.ft_toeplitz_matvec.argtypes = [P, P, U64, U64, P, P]
        L.ft_block_matvec.argtypes = [P, P, U64, U64, C.c_double, P, P]
        L.ft_set_exchange.argtypes = [P, EXCHANGE_FN, P, P, P]
        L.ft_plan_get_info.argtypes = [P, C.POINTER(_Info)]
        L.ft_column.argtypes = [P, U64, P]
        L.ft_assemble_rhs.argtypes = [P, FORCING_FN, INITIAL_FN, INITIAL_FN, P, P]
        L.ft_assemble_rhs_grid.argtypes = [P, P, P, P, P]
        L.ft_assemble_rhs_modes.argtypes = [P, I, P, P, P, P, P, P, P]
        L.ft_solve_fast.argtypes = [P, P, P, C.POINTER(_Report)]
        L.ft_solve_direct.argtypes = [P, P, P, C.POINTER(_Report)]
        L.ft_solve_fast_modes.argtypes = [P, I, P, P, P, P, P, P, P, C.POINTER(_Report)]
        L.ft_apply.argtypes = [P, P, P]
        L.ft_residual.argtypes = [P, P, P, P, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ft_nccl_unique_id.argtypes = [P]
        L.ft_nccl_init.argtypes = [P, P, I, I]
        L.ft_p2p_handle.argtypes = [P, P]
        L.ft_p2p_connect.argtypes = [P, P]
        L.ft_set_stream.argtypes = [P, P]
        L.ft_profile_fast.argtypes = [P, P, P, C.POINTER(_OpTime), U64, C.POINTER(U64)]
        L.ft_schedule.argtypes = [U64, U64, C.POINTER(_OpTime), U64, C.POINTER(U64)]
        L.ft_last_error.restype = C.c_char_p
        L.ft_destroy.argtypes = [P]
        L.ft_destroy.restype = None
        for name in ABI_SYMBOLS:
            if name not in ("ft_last_error", "ft_destroy"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().ft_last_error().decode()
        if rc == -1:
            raise InvalidArgument(rc, msg)
        if rc == -2:
            raise DomainError(rc, msg)
        raise FractimeError(rc, msg)


def _ptr(a, count: Optional[int] = None, what: str = "buffer") -> int:
    """Device pointer of a torch tensor or host pointer of a numpy array, after
    checking dtype (float64), contiguity and, when given, the element count --
    the C ABI takes plain pointers, so a wrong buffer would be written out of
    bounds instead of failing."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64:
            raise InvalidArgument(-1, f"{what}: float64 expected, got {a.dtype}")
        if not a.flags.c_contiguous:
            raise InvalidArgument(-1, f"{what}: C-contiguous array expected")
        if count is not None and a.size != count:
            raise InvalidArgument(-1, f"{what}: {count} elements expected, got {a.size}")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        import torch

        if a.dtype != torch.float64:
            raise InvalidArgument(-1, f"{what}: torch.float64 expected, got {a.dtype}")
        if not a.is_contiguous():
            raise InvalidArgument(-1, f"{what}: contiguous tensor expected")
        if count is not None and a.numel() != count:
            raise InvalidArgument(-1, f"{what}: {count} elements expected, got {a.numel()}")
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)}")


@dataclass
class ProblemSpec:
    """Reference ProblemSpec (schemes.hpp:191-205).  Callbacks take (x, t) / (x)."""

    scheme: SchemeId = SchemeId.Diffusion
    gamma: float = 0.5
    time_steps: int = 2
    space_cells: int = 0
    time_length: float = 1.0
    space_length: float = 1.0
    forcing: Optional[Callable[[float, float], float]] = None
    initial_u0: Optional[Callable[[float], float]] = None
    initial_phi: Optional[Callable[[float], float]] = None
    exact: Optional[Callable[[float, float], float]] = None

    def tau(self) -> float:
        return self.time_length / self.time_steps

    def h(self) -> float:
        return self.space_length / self.space_cells if self.space_cells else 0.0

    def _c(self) -> _Problem:
        return _Problem(int(self.scheme), float(self.gamma), int(self.time_steps),
                        int(self.space_cells), float(self.time_length), float(self.space_length))


@dataclass
class SolutionGrid:
    """Reference SolutionGrid (schemes.hpp:213-223): node-major values."""

    scheme: SchemeId
    tau: float
    h: float
    time_steps: int
    space_cells: int
    values: np.ndarray

    def at(self, i: int, n: int) -> float:
        return float(self.values[(i - 1) * self.time_steps + (n - 1)])


@dataclass
class SolveReport:
    method: str = ""
    iterations: int = 0
    residual: float = 0.0
    seconds: float = 0.0
    device_ms: float = 0.0
    kernel_launches: int = 0


@dataclass
class SchemeSolution:
    grid: SolutionGrid
    report: SolveReport = field(default_factory=SolveReport)


class Plan:
    """A device-resident solver plan (ft_setup / ft_setup_batch; Plan.toeplitz for
    ft_setup_toeplitz)."""

    def __init__(self, problems, rhs_mode: int = FT_RHS_REFERENCE, near_field: int = 0,
                 device: int = -1, partition=None, _handle=None, report_residual: bool = False):
        if _handle is not None:
            self.specs = []
            h = _handle
        else:
            if isinstance(problems, ProblemSpec):
                problems = [problems]
            self.specs = list(problems)
            arr = (_Problem * len(self.specs))(*[p._c() for p in self.specs])
            opt = _Options(rhs_mode, near_field, device, 1 if report_residual else 0)
            h = C.c_void_p()
            if partition is None:
                _check(lib().ft_setup_batch(arr, len(self.specs), C.byref(opt), C.byref(h)))
            else:
                rank, world = partition
                _check(lib().ft_setup_partitioned(arr, C.byref(opt), rank, world, C.byref(h)))
        self._h = h
        self._device = device
        info = _Info()
        _check(lib().ft_plan_get_info(self._h, C.byref(info)))
        self.info = info
        self.B = int(info.problems)
        self.nodes = int(info.local_nodes)        # rows per problem held by this plan
        self.global_nodes = int(info.nodes)
        self.node_begin = int(info.node_begin)
        self.N = int(info.time_steps)

    @classmethod
    def toeplitz(cls, first_cols, device: int = -1) -> "Plan":
        """Lower-triangular Toeplitz systems with the caller's first columns
        ([count][n] or [n]); ToeplitzOperator::lower_triangular +
        lower_toeplitz_forward_solve (toeplitz.cpp:169-186).  Buffers are [count][n]."""
        cols = np.atleast_2d(np.ascontiguousarray(first_cols, dtype=np.float64))
        opt = _Options(0, 0, device, 0)
        h = C.c_void_p()
        _check(lib().ft_setup_toeplitz(cols.ctypes.data, cols.shape[1], cols.shape[0], C.byref(opt), C.byref(h)))
        return cls(None, _handle=h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.ft_destroy(h)
            self._h = None

    @property
    def shape(self):
        return (self.B * self.nodes, self.N)

    def column(self, problem: int = 0) -> np.ndarray:
        out = np.empty(self.N)
        _check(lib().ft_column(self._h, problem, out.ctypes.data))
        return out

    def assemble_rhs(self, forcing, u0=None, phi=None) -> np.ndarray:
        """Host callbacks, evaluated at the reference's points (slow; small sizes)."""
        f = FORCING_FN(lambda x, t, _u: forcing(x, t))
        g = INITIAL_FN(lambda x, _u: u0(x)) if u0 else C.cast(None, INITIAL_FN)
        q = INITIAL_FN(lambda x, _u: phi(x)) if phi else C.cast(None, INITIAL_FN)
        out = np.empty(self.shape)
        _check(lib().ft_assemble_rhs(self._h, f, g, q, None, out.ctypes.data))
        return out

    def assemble_rhs_grid(self, F: np.ndarray, u0=None, phi=None) -> np.ndarray:
        F = np.ascontiguousarray(F, dtype=np.float64)
        u0 = None if u0 is None else np.ascontiguousarray(u0, dtype=np.float64)
        phi = None if phi is None else np.ascontiguousarray(phi, dtype=np.float64)
        out = np.empty(self.shape)
        _check(lib().ft_assemble_rhs_grid(self._h, _ptr(F), _ptr(u0), _ptr(phi), out.ctypes.data))
        return out

    def _mode_args(self, a, k, p, trig, u0amp, phiamp):
        k = np.ascontiguousarray(k, dtype=np.float64).reshape(-1)
        nm = k.size
        a = np.ascontiguousarray(a, dtype=np.float64)
        p = np.ascontiguousarray(p, dtype=np.float64)
        trig = np.ascontiguousarray(trig, dtype=np.int32).reshape(-1)
        for name, arr in (("a", a), ("p", p)):
            if arr.size != self.B * nm:
                raise InvalidArgument(-1, f"{name}: shape ({self.B}, {nm}) expected, got {arr.shape}")
        if trig.size != nm:
            raise InvalidArgument(-1, f"trig: {nm} entries expected, got {trig.size}")
        u0amp = None if u0amp is None else np.ascontiguousarray(u0amp, dtype=np.float64).reshape(-1)
        phiamp = None if phiamp is None else np.ascontiguousarray(phiamp, dtype=np.float64).reshape(-1)
        for name, arr in (("u0amp", u0amp), ("phiamp", phiamp)):
            if arr is not None and arr.size != self.B:
                raise InvalidArgument(-1, f"{name}: {self.B} entries expected, got {arr.size}")
        return a, k, p, trig, u0amp, phiamp

    def assemble_rhs_modes(self, out, a, k, p, trig, u0amp=None, phiamp=None):
        """Device generation of a separable forcing into the device buffer `out`."""
        a, k, p, trig, u0amp, phiamp = self._mode_args(a, k, p, trig, u0amp, phiamp)
        self._check_device(out, "rhs")
        _check(lib().ft_assemble_rhs_modes(self._h, len(k), a.ctypes.data, k.ctypes.data,
                                           p.ctypes.data, trig.ctypes.data,
                                           None if u0amp is None else u0amp.ctypes.data,
                                           None if phiamp is None else phiamp.ctypes.data,
                                           _ptr(out, self.shape[0] * self.shape[1], "rhs")))
        return out

    def _check_device(self, buf, what):
        if hasattr(buf, "is_cuda") and buf.is_cuda and int(self.info_device()) >= 0:
            if buf.device.index != self.info_device():
                raise InvalidArgument(-1, f"{what}: tensor on cuda:{buf.device.index}, plan on cuda:{self.info_device()}")

    def info_device(self) -> int:
        return getattr(self, "_device", -1)

    def _solve(self, fn, rhs, out):
        if out is None:
            out = np.empty(self.shape) if isinstance(rhs, np.ndarray) else rhs.new_empty(self.shape)
        n = self.shape[0] * self.shape[1]
        self._check_device(rhs, "rhs")
        self._check_device(out, "u")
        rep = _Report()
        _check(fn(self._h, _ptr(rhs, n, "rhs"), _ptr(out, n, "u"), C.byref(rep)))
        report = SolveReport(rep.method.decode(), rep.iterations, rep.residual, rep.seconds,
                             rep.device_ms, rep.kernel_launches)
        return out, report

    def set_stream(self, stream_handle: int) -> None:
        """Run on a caller's CUDA stream (e.g. torch.cuda.current_stream().cuda_stream)."""
        _check(lib().ft_set_stream(self._h, stream_handle))

    def profile_fast(self, rhs, out):
        """Per-launch device times of one fast solve (device buffers)."""
        cap = 4 * (self.N // 8 + 16)
        arr = (_OpTime * cap)()
        cnt = C.c_uint64(0)
        _check(lib().ft_profile_fast(self._h, _ptr(rhs), _ptr(out), arr, cap, C.byref(cnt)))
        return [dict(kind=arr[i].kind, level=arr[i].level, t0=arr[i].t0, len=arr[i].len,
                     bytes=arr[i].bytes, ms=arr[i].ms) for i in range(min(cnt.value, cap))]

    def nccl_init(self, unique_id: bytes, rank: int = 0, world: int = 1) -> None:
        """Bind the per-leaf carry all-gather to ncclAllGather on the plan's stream (collective:
        every rank calls it with rank 0's `nccl_unique_id()`); the solve then replays as one
        CUDA graph with the collectives inside."""
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _check(lib().ft_nccl_init(self._h, buf, rank, world))

    def apply(self, x, out=None):
        """y = A x with the plan's system matrix (the reference's block operator, applied
        through the plan's FFT history products); x, out: both device tensors or both host arrays."""
        if out is None:
            out = np.empty(self.shape) if isinstance(x, np.ndarray) else x.new_empty(self.shape)
        n = self.shape[0] * self.shape[1]
        self._check_device(x, "x")
        self._check_device(out, "y")
        _check(lib().ft_apply(self._h, _ptr(x, n, "x"), _ptr(out, n, "y")))
        return out

    def residual(self, rhs, u, work=None):
        """(max |A u - rhs|, max |rhs|) on the device."""
        n = self.shape[0] * self.shape[1]
        r, m = C.c_double(0.0), C.c_double(0.0)
        _check(lib().ft_residual(self._h, _ptr(rhs, n, "rhs"), _ptr(u, n, "u"),
                                 None if work is None else _ptr(work, n, "work"), C.byref(r), C.byref(m)))
        return r.value, m.value

    def solve_fast(self, rhs, out=None):
        return self._solve(lib().ft_solve_fast, rhs, out)

    def solve_direct(self, rhs, out=None):
        return self._solve(lib().ft_solve_direct, rhs, out)

    def solve_fast_modes(self, out, a, k, p, trig, u0amp=None, phiamp=None):
        """Fast solve with the separable forcing of assemble_rhs_modes generated
        inside the leaves (the right-hand side is never materialised); `out`
        (host or device, [rows][N]) receives U."""
        a, k, p, trig, u0amp, phiamp = self._mode_args(a, k, p, trig, u0amp, phiamp)
        self._check_device(out, "u")
        rep = _Report()
        _check(lib().ft_solve_fast_modes(self._h, len(k), a.ctypes.data, k.ctypes.data, p.ctypes.data,
                                         trig.ctypes.data, None if u0amp is None else u0amp.ctypes.data,
                                         None if phiamp is None else phiamp.ctypes.data,
                                         _ptr(out, self.shape[0] * self.shape[1], "u"), C.byref(rep)))
        return out, SolveReport(rep.method.decode(), rep.iterations, rep.residual, rep.seconds,
                                rep.device_ms, rep.kernel_launches)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the solver's run-time NCCL binding (rank 0; ship to all ranks)."""
    buf = (C.c_ubyte * 128)()
    _check(lib().ft_nccl_unique_id(buf))
    return bytes(buf)


def schedule(time_steps: int, leaf: int = 32):
    """The divide-and-conquer launch schedule (host-only, no GPU needed)."""
    cap = 2 * (time_steps // leaf + 2)
    arr = (_OpTime * cap)()
    cnt = C.c_uint64(0)
    _check(lib().ft_schedule(time_steps, leaf, arr, cap, C.byref(cnt)))
    return [dict(kind=arr[i].kind, level=arr[i].level, t0=arr[i].t0, len=arr[i].len)
            for i in range(cnt.value)]


def toeplitz_matvec(first_col, x, first_row=None):
    """y = T x for one vector [n] or a batch [count][n] (reference toeplitz_matvec,
    toeplitz.cpp:98-115; first_row None = lower triangular).  numpy or torch
    (host or CUDA) arrays; returns the same kind."""
    col = np.ascontiguousarray(first_col, dtype=np.float64)
    row = None if first_row is None else np.ascontiguousarray(first_row, dtype=np.float64)
    n = col.shape[0]
    count = int(np.prod(x.shape)) // n
    y = np.empty_like(x) if isinstance(x, np.ndarray) else x.new_empty(x.shape)
    _check(lib().ft_toeplitz_matvec(col.ctypes.data, None if row is None else row.ctypes.data, n, count,
                                    _ptr(x), _ptr(y)))
    return y


def block_matvec(first_col, m_blocks: int, off_scale: float, x, first_row=None):
    """Block tridiagonal Toeplitz operator apply (reference block_matvec,
    toeplitz.cpp:150-167); x is [m_blocks * n] or [m_blocks][n]."""
    col = np.ascontiguousarray(first_col, dtype=np.float64)
    row = None if first_row is None else np.ascontiguousarray(first_row, dtype=np.float64)
    y = np.empty_like(x) if isinstance(x, np.ndarray) else x.new_empty(x.shape)
    _check(lib().ft_block_matvec(col.ctypes.data, None if row is None else row.ctypes.data, col.shape[0], m_blocks,
                                 float(off_scale), _ptr(x), _ptr(y)))
    return y


def lower_toeplitz_solve(first_col, b, method: SolveMethod = SolveMethod.Fast):
    """x with T x = b, T lower-triangular Toeplitz (reference
    lower_toeplitz_forward_solve, toeplitz.cpp:169-186) -- the D&C (Fast) or
    the reference's substitution order (Direct)."""
    plan = Plan.toeplitz(first_col)
    bb = np.ascontiguousarray(b, dtype=np.float64).reshape(plan.shape) if isinstance(b, np.ndarray) else b
    x, _ = (plan.solve_fast if method == SolveMethod.Fast else plan.solve_direct)(bb)
    return x.reshape(np.shape(b)) if isinstance(b, np.ndarray) else x


def solve(spec: ProblemSpec, method: SolveMethod = SolveMethod.Fast, rhs_mode: int = 0) -> SchemeSolution:
    """Reference solve(spec, method, cfg) (schemes.cpp:481-489) on the GPU."""
    t0 = time.perf_counter()
    plan = Plan(spec, rhs_mode=rhs_mode)
    rhs = plan.assemble_rhs(spec.forcing, spec.initial_u0, spec.initial_phi)
    if method == SolveMethod.Fast:
        u, rep = plan.solve_fast(rhs)
    else:
        u, rep = plan.solve_direct(rhs)
    rep.seconds = time.perf_counter() - t0
    grid = SolutionGrid(spec.scheme, spec.tau(), spec.h(), spec.time_steps, spec.space_cells,
                        u.reshape(-1))
    return SchemeSolution(grid, rep)


def l2_error(grid: SolutionGrid, spec: ProblemSpec) -> float:
    """Reference l2_error (schemes.cpp:525-542); the ODE variant uses the one-sided
    scheme's nodes n = 1..N."""
    if spec.exact is None:
        raise InvalidArgument(-1, "l2_error: spec has no exact solution")
    acc = 0.0
    if grid.scheme == SchemeId.Ode:
        for n in range(1, grid.time_steps + 1):
            e = grid.values[n - 1] - spec.exact(0.0, n * grid.tau)
            acc += grid.tau * e * e
    else:
        tf = grid.time_steps * grid.tau
        for i in range(1, grid.space_cells):
            e = grid.at(i, grid.time_steps) - spec.exact(i * grid.h, tf)
            acc += grid.h * e * e
    return math.sqrt(acc)


__all__ = ["FractimeError", "InvalidArgument", "DomainError", "SchemeId", "SolveMethod", "ProblemSpec",
           "SolutionGrid", "SolveReport", "SchemeSolution", "Plan", "solve", "l2_error", "lib",
           "nccl_unique_id", "ABI_SYMBOLS", "FT_RHS_REFERENCE", "FT_RHS_CORRECTED_N1", "schedule"]
