"""The A/B switches of the fast path keep their alternative kernels correct.

Each switch is read once per process (a function static in the library), so
every variant runs in its own interpreter: a wide config-4-shaped plan (8 slabs:
the cooperative slab leaf with the level-0 products folded in) and a config-2
shaped plan (every single-CTA FFT level up to n = 4096), fast solve against the
on-device reference-order march (ft_solve_direct, pinned bitwise to the CPU
oracle by tests/test_gpu_scale.py).  Tolerance (north_star): 1e-10 relative.

  default        leaf pairs (leaf_pair), lean slab leaf, mp1g_kernel
  FT_NO_PAIR=1   one cooperative kernel per leaf (leaf_fused, level-0 product from global memory)
  FT_NO_LEAN=1   the generic slab-leaf instantiation (and no pairs)
  FT_MP1P=1      persistent TMA-staged FFT levels (mp1p_kernel: cp.async.bulk + mbarrier)
  FT_MP8=0x1f00  radix-8 high-occupancy FFT levels (mp8_kernel, n = 256 .. 4096) and their spectra
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys; sys.path.insert(0, %r)
import torch
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
worst = 0.0
for cid, kw in ((4, dict(time_steps=512, cells=3587)), (2, dict(time_steps=4096))):
    w = W.config(cid, **kw)
    plan = ft.Plan(w.specs, device=0)
    R = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    plan.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig, w.u0amp, w.phiamp)
    uf, rep = plan.solve_fast(R)
    ud, _ = plan.solve_direct(R)
    err = ((uf - ud).abs().max() / ud.abs().max()).item()
    print(f"cfg{cid} launches={rep.kernel_launches} shape={tuple(plan.shape)} fast-vs-direct-march={err:.3e}")
    worst = max(worst, err)
print("WORST", worst)
sys.exit(0 if worst <= 1e-10 else 1)
""" % str(ROOT)


def _run(env_extra):
    env = dict(os.environ)
    for k in ("FT_NO_PAIR", "FT_NO_LEAN", "FT_MP1P", "FT_MP8"):
        env.pop(k, None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    return r.stdout


def _launches(out, cid):
    line = next(l for l in out.splitlines() if l.startswith(f"cfg{cid} "))
    return int(line.split("launches=")[1].split()[0])


def test_default_uses_leaf_pairs():
    out = _run({})
    # 16 leaves as 8 pair kernels + the 7 products above level 0
    assert _launches(out, 4) == 15, out


def test_no_pair_variant():
    out = _run({"FT_NO_PAIR": "1"})
    assert _launches(out, 4) == 23, out  # 16 leaf kernels + 7 products (level 0 folded into the leaves)


def test_generic_slab_leaf_variant():
    _run({"FT_NO_LEAN": "1"})


def test_tma_staged_fft_levels_variant():
    _run({"FT_MP1P": "1"})


def test_radix8_high_occupancy_fft_levels_variant():
    _run({"FT_MP8": "0x1f00"})
