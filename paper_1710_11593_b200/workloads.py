"""The BASELINE.json configurations as solver workloads.

Each workload is a list of ProblemSpec-like parameters plus a separable
forcing  f_b(x,t) = sum_j a[b,j] trig_j(k_j pi x) t^p[b,j]  and initial-data
amplitudes (u0 = amp * sin(pi x), phi likewise; the ODE uses u0 = amp).
Seeded draws use splitmix64 with master seed 0x171011593, stream = master
XOR config id; uniforms ((x >> 11) + 0.5) * 2^-53; normals by Box-Muller
(cosine branch).  The oracle (oracle/oracle.c) implements the same generator;
tests/test_workloads.py checks they agree.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import ProblemSpec, SchemeId

MASTER_SEED = 0x171011593
_M64 = (1 << 64) - 1


class SplitMix64:
    def __init__(self, seed: int):
        self.state = seed & _M64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return ((self.next() >> 11) + 0.5) * 2.0 ** -53

    def normal(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * 3.14159265358979323846 * u2)


@dataclass
class Workload:
    name: str
    specs: List[ProblemSpec]
    a: np.ndarray        # [B, nmodes]
    k: np.ndarray        # [nmodes]
    p: np.ndarray        # [B, nmodes]
    trig: np.ndarray     # [nmodes] 0 sin, 1 cos, 2 const
    u0amp: Optional[np.ndarray]
    phiamp: Optional[np.ndarray]
    exact: Optional[str] = None   # closed form of u for error reports

    @property
    def B(self) -> int:
        return len(self.specs)

    @property
    def nodes(self) -> int:
        s = self.specs[0]
        return 1 if s.scheme == SchemeId.Ode else s.space_cells - 1

    @property
    def N(self) -> int:
        return self.specs[0].time_steps

    @property
    def unknowns(self) -> int:
        return self.B * self.nodes * self.N


def example(eid: int, gamma: float, e: int) -> Workload:
    """The reference's manufactured Examples 2, 3 and 4 (proj/src/harness.cpp:58-86)
    at h = tau = 2^-e, as used by its acceptance tables (acceptance.cpp:62-90)."""
    n = 1 << e
    if eid == 2:  # transport (Scheme 2), u = t sin(pi x), forcing at ((i - 1/2) h, n tau)
        spec = ProblemSpec(SchemeId.Hyperbolic, gamma, n, n, 1.0, 1.0)
        a = np.array([[1.0 / math.gamma(2.0 - gamma), math.pi]])
        p = np.array([[1.0 - gamma, 1.0]])
        return Workload(f"example2-e{e}", [spec], a, np.array([1.0, 1.0]), p, np.array([0, 1]), None, None,
                        "t sin(pi x)")
    if eid == 4:  # diffusion, u = t^3 sin(pi x)
        spec = ProblemSpec(SchemeId.Diffusion, gamma, n, n, 1.0, 1.0)
        a = np.array([[6.0 / math.gamma(4.0 - gamma), math.pi ** 2]])
        p = np.array([[3.0 - gamma, 3.0]])
        return Workload(f"example4-e{e}", [spec], a, np.array([1.0, 1.0]), p, np.array([0, 0]), None, None,
                        "t^3 sin(pi x)")
    if eid == 3:  # wave, u = t^3 x (1 - x)
        spec = ProblemSpec(SchemeId.DiffusionWave, gamma, n, n, 1.0, 1.0)
        a = np.array([[6.0 / math.gamma(4.0 - gamma), 1.0]])
        p = np.array([[3.0 - gamma, 3.0]])
        return Workload(f"example3-e{e}", [spec], a, np.array([1.0, 1.0]), p, np.array([3, 4]), None, None,
                        "t^3 x (1-x)")
    raise ValueError(eid)


def transport(gamma: float, time_steps: int, cells: int, u0amp: Optional[float] = None) -> Workload:
    """Scheme 2 (transport) test problem: Example 2's forcing (harness.cpp:58-67)
    on an arbitrary mesh, optionally with u0 = u0amp sin(pi x) to exercise the
    initial-data term of Scheme2Rhs (schemes.cpp:183-187)."""
    w = example(2, gamma, 1)
    s = w.specs[0]
    s.time_steps, s.space_cells = time_steps, cells
    w.name = f"transport-g{gamma}-n{time_steps}-c{cells}"
    if u0amp is not None:
        w.u0amp = np.array([float(u0amp)])
        w.exact = None
    return w


def exact_final(w: Workload) -> np.ndarray:
    """Exact solution at t = T on the interior nodes (for the examples / configs)."""
    s = w.specs[0]
    x = np.arange(1, s.space_cells) * s.h()
    t = s.time_length
    if w.exact == "t sin(pi x)":
        return t * np.sin(np.pi * x)
    if w.exact == "t^3 sin(pi x)":
        return t ** 3 * np.sin(np.pi * x)
    if w.exact == "t^3 x (1-x)":
        return t ** 3 * x * (1 - x)
    if w.exact == "(t^2+1) sin(pi x)":
        return (t ** 2 + 1) * np.sin(np.pi * x)
    if w.exact == "(t^3+t+1) sin(pi x)":
        return (t ** 3 + t + 1) * np.sin(np.pi * x)
    raise ValueError(w.exact)


def l2_final(w: Workload, U: np.ndarray) -> float:
    """Reference l2_error (schemes.cpp:525-542): final-time spatial L2 norm."""
    s = w.specs[0]
    e = U[:, -1] - exact_final(w)
    return float(np.sqrt(np.sum(s.h() * e * e)))


def config(cid: int, time_steps: Optional[int] = None, cells: Optional[int] = None,
           batch: Optional[int] = None) -> Workload:
    """BASELINE.json configs[cid-1].  time_steps < N gives the time-prefix
    variant (time_length = N'/N so tau stays 1/N exactly);
    cells overrides M+1 (reduced-M variant)."""
    if cid == 1:
        g, N = 0.5, 4096
        Np = time_steps or N
        spec = ProblemSpec(SchemeId.Ode, g, Np, 0, Np / N, 1.0)
        a = np.array([[2.0 / math.gamma(3.0 - g), 1.0, 1.0]])
        p = np.array([[2.0 - g, 2.0, 0.0]])
        return Workload("cfg1-ode", [spec], a, np.array([1.0, 1.0, 1.0]), p, np.array([2, 2, 2]),
                        np.array([1.0]), None, "t^2+1")
    if cid == 2:
        g, N, c = 0.7, 16384, (cells or 257)
        Np = time_steps or N
        spec = ProblemSpec(SchemeId.Diffusion, g, Np, c, Np / N, 1.0)
        a = np.array([[2.0 / math.gamma(3.0 - g), math.pi ** 2, math.pi ** 2]])
        p = np.array([[2.0 - g, 2.0, 0.0]])
        return Workload("cfg2-diffusion", [spec], a, np.array([1.0, 1.0, 1.0]), p, np.array([0, 0, 0]),
                        np.array([1.0]), None, "(t^2+1) sin(pi x)")
    if cid == 3:
        g, N, c = 1.5, 65536, (cells or 1025)
        Np = time_steps or N
        spec = ProblemSpec(SchemeId.DiffusionWave, g, Np, c, Np / N, c / 1025.0 if cells else 1.0)
        a = np.array([[6.0 / math.gamma(4.0 - g), math.pi, math.pi, math.pi]])
        p = np.array([[3.0 - g, 3.0, 1.0, 0.0]])
        return Workload("cfg3-wave", [spec], a, np.array([1.0, 1.0, 1.0, 1.0]), p,
                        np.array([0, 1, 1, 1]), np.array([1.0]), np.array([1.0]), "(t^3+t+1) sin(pi x)")
    if cid == 4:
        g, N, c = 0.3, 65536, (cells or 65537)
        Np = time_steps or N
        rng = SplitMix64(MASTER_SEED ^ 4)
        a, p = [], []
        for _ in range(8):
            a.append(rng.normal())
            p.append(1.0 + 2.0 * rng.uniform())
        spec = ProblemSpec(SchemeId.Diffusion, g, Np, c, Np / N, 1.0)
        return Workload("cfg4-diffusion-large", [spec], np.array([a]), np.arange(1.0, 9.0),
                        np.array([p]), np.zeros(8, dtype=np.int32), None, None)
    if cid == 5:
        N, c = 32768, (cells or 513)
        Np = time_steps or N
        nb = 64
        rng = SplitMix64(MASTER_SEED ^ 5)
        specs, A, Pw = [], [], []
        for _ in range(nb):
            g = 0.1 + 0.8 * rng.uniform()
            pe = 1.0 + rng.uniform()
            aa = [rng.normal() for _ in range(4)]
            specs.append(ProblemSpec(SchemeId.Diffusion, g, Np, c, Np / N, 1.0))
            A.append(aa)
            Pw.append([pe] * 4)
        nb_used = batch or nb
        return Workload("cfg5-batch", specs[:nb_used], np.array(A[:nb_used]), np.arange(1.0, 5.0),
                        np.array(Pw[:nb_used]), np.zeros(4, dtype=np.int32), np.ones(nb_used), None)
    raise ValueError(cid)
