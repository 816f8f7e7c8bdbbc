#!/usr/bin/env python3
"""Generate tests/golden/golden.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference and oracle/_ref built by
oracle/build_ref.sh).  Everything in the fixture is produced by the reference
itself (its weights, its direct and fast solvers through its public API) or
parsed from the reference's own acceptance test (frozen paper tables); inputs
are the seeded synthetic workloads of paper_1710_11593_b200.workloads sampled
by the oracle's glibc forcing generator.

    python tests/golden/make_golden.py
"""
import json
import re
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1710_11593_b200 import workloads as W  # noqa: E402

REF_ACCEPT = Path("/root/reference/proj/tests/acceptance.cpp")


def parse_tables():
    """kDiffusionReference / kWaveReference from the reference acceptance test."""
    src = REF_ACCEPT.read_text()
    out = {}
    for name in ("kDiffusionReference", "kWaveReference", "kTransportReference"):
        body = src[src.index(name):]
        body = body[:body.index("};")]
        cols = []
        for m in re.finditer(r"\{([0-9.]+),\s*\{([^}]*)\},\s*\{([^}]*)\}\}", body):
            cols.append({"gamma": float(m.group(1)),
                         "errors": [float(x) for x in m.group(2).split(",")],
                         "rates": [float(x) for x in m.group(3).split(",")]})
        out[name] = cols
    return out


CASES = [  # (name, config, kwargs) -- small enough for the reference direct path
    ("cfg1_n256", 1, dict(time_steps=256)),
    ("cfg2_m16_n128", 2, dict(time_steps=128, cells=17)),
    ("cfg2_m31_n100", 2, dict(time_steps=100, cells=32)),
    ("cfg3_m16_n128", 3, dict(time_steps=128, cells=17)),
    ("cfg4_m32_n64", 4, dict(time_steps=64, cells=33)),
    ("cfg4_m4096_n16", 4, dict(time_steps=16, cells=4097)),
    ("s2_g0.5_n16_m8", "transport", dict(gamma=0.5, time_steps=16, cells=8)),
    ("s2_g0.3_n64_m33_u0", "transport", dict(gamma=0.3, time_steps=64, cells=33, u0amp=1.0)),
    ("s2_g0.9_n100_m20_u0", "transport", dict(gamma=0.9, time_steps=100, cells=20, u0amp=-0.7)),
]


def case_workload(cid, kw):
    return W.transport(**kw) if cid == "transport" else W.config(cid, **kw)


def main():
    L = oracle.rlib()
    if L is None:
        raise SystemExit("build the reference first: bash oracle/build_ref.sh")
    data = {}
    # weights known-answer values (reference weights.cpp)
    for kind, g, n in ((0, 0.5, 4), (1, 1.5, 3), (0, 0.3, 2000), (1, 1.7, 2000)):
        w = np.empty(n)
        assert L.ref_weights(kind, g, n, w.ctypes.data) == 0
        data[f"weights_{kind}_{g}_{n}"] = w
    data["power_step_1e9_0.5"] = np.array([L.ref_power_step(1000000000, 0.5)])
    # solutions through the reference's public solve() / Toeplitz API
    for name, cid, kw in CASES:
        w = case_workload(cid, kw)
        s = w.specs[0]
        F = oracle.forcing_grid(w)
        u0 = oracle.initial_grid(w, w.u0amp)
        phi = oracle.initial_grid(w, w.phiamp)
        data[f"{name}_F"] = F
        if u0 is not None:
            data[f"{name}_u0"] = u0
        if phi is not None:
            data[f"{name}_phi"] = phi
        if cid == 1:
            N = s.time_steps
            col = np.empty(N)
            assert L.ref_ode_column(s.gamma, N, s.time_length, col.ctypes.data) == 0
            R = oracle.rhs(w, F, u0)
            U = np.empty(N)
            assert L.ref_forward_solve(col.ctypes.data, R.ctypes.data, N, U.ctypes.data) == 0
            data[f"{name}_col"] = col
            data[f"{name}_direct"] = U.reshape(1, N)
        else:
            U, _, _ = oracle.ref_solve(s, "direct", F, u0, phi)
            data[f"{name}_direct"] = U
            # the reference's own setup: first column(s) and (Scheme 4) the assembled RHS
            col, col2, _, R = oracle.ref_setup(s, F, u0)
            data[f"{name}_col"] = col
            if col2 is not None:
                data[f"{name}_col2"] = col2
            if R is not None:
                data[f"{name}_rhs"] = R
    np.savez_compressed(Path(__file__).with_name("golden.npz"), **data)
    Path(__file__).with_name("tables.json").write_text(json.dumps(parse_tables(), indent=1))
    print("wrote", len(data), "arrays")


if __name__ == "__main__":
    main()
