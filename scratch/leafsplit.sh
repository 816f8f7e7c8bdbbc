for d in 0 1 2 3; do FT_LEAF_DBG=$d python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
wl=W.config(4, time_steps=4096); plan=ft.Plan(wl.specs)
rhs=torch.empty(plan.shape,dtype=torch.float64,device='cuda'); u=torch.empty_like(rhs)
plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
plan.solve_fast(rhs,u); ops=plan.profile_fast(rhs,u)
lf=[o for o in ops if o['kind']==0]
print('dbg', $d, 'leaf us/leaf', 1e3*sum(o['ms'] for o in lf)/len(lf))
"; done
