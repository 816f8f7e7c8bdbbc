import sys, ctypes as C; sys.path.insert(0,'.')
import torch, numpy as np, paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
wl=W.config(4, time_steps=4096); plan=ft.Plan(wl.specs)
rhs=torch.empty(plan.shape,dtype=torch.float64,device='cuda'); u=torch.empty_like(rhs)
plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
plan.solve_fast(rhs,u)
c=(C.c_longlong*16)(); ft.lib().ft_debug_leaf_clocks.argtypes=[C.c_void_p, C.c_void_p]
assert ft.lib().ft_debug_leaf_clocks(plan._h, C.addressof(c))==0
v=list(c)
print("phase1 [cycles]: stage+setup", v[9]-v[8], " steps", v[10]-v[9], " store", v[11]-v[10])
if len(sys.argv) > 1 and sys.argv[1] == "ws":
    print("correct_ws: load c0+h", v[1]-v[0], " phase2", v[2]-v[1], " join", v[3]-v[2], " phase3", v[4]-v[3], " store", v[5]-v[4])
else:
    print("correct: load c0+h", v[1]-v[0], " phase2(+staging x)", v[2]-v[1], " phase3", v[3]-v[2], " store", v[4]-v[3])
if len(sys.argv) > 1 and sys.argv[1] == "ws":
    b = v[6]
    print("scan warp step 5 (from sync2 release): loads+shfl scan", v[7]-b, " bar3#1", v[12]-b, " crosswarp+bar3#2", v[13]-b,
          " EL/ER+STS", v[14]-b, " | response sync1 release", v[15]-b)
