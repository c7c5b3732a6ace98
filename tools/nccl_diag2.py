"""Bench-like loop on the one-rank NCCL communicator: several steps, then timing mode, then destroy."""
import faulthandler
import sys
import time

import numpy as np
import torch

faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, ".")
from paper_2303_03398_b200 import inputs, maspcg  # noqa: E402

path = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = inputs.make_problem("c3", shape=(150, 300, 64))
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
kr, kt, kp, s, f, x0 = (T(a) for a in (p.kr, p.kt, p.kp, p.s, p.f, p.x0))
S = maspcg.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf, force_comm=True)
S.set_option(maspcg.OPT_PATH, path)
x = torch.empty_like(x0)
for it in range(6):
    if it == 3:
        S.set_option(maspcg.OPT_TIMING, 2)
    t = time.time()
    S.set_grid(p.rf, p.tf, p.pf)
    print("step", it, "grid", flush=True)
    S.set_coefficients(kr, kt, kp, s)
    print("step", it, "coef", flush=True)
    S.set_bc_r(p.bc_in, None, p.bc_out, None)
    x.copy_(x0)
    st, info, hist = S.solve(f, x, 1e-10, 20000)
    torch.cuda.synchronize()
    print("step", it, st, info["iters"], round(time.time() - t, 3), flush=True)
S.close()
print("closed", flush=True)
