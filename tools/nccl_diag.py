"""Diagnose the one-rank NCCL communicator path at growing plane sizes (each case in its own process)."""
import json
import os
import subprocess
import sys
import time

CASE = r'''
import sys, time, faulthandler, numpy as np, torch
faulthandler.dump_traceback_later(50, exit=True)
sys.path.insert(0, ".")
from paper_2303_03398_b200 import inputs, maspcg
name, shape, graphs, path, maxit = sys.argv[1], eval(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
p = inputs.make_problem(name, shape=shape)
S = maspcg.solver_for_problem(p, force_comm=True)
S.set_option(maspcg.OPT_USE_GRAPHS, graphs)
S.set_option(maspcg.OPT_PATH, path)
x = torch.from_numpy(p.x0.copy()).cuda()
t = time.time()
st, info, hist = S.solve(torch.from_numpy(p.f).cuda(), x, 0.0, maxit)
torch.cuda.synchronize()
print("OK", name, shape, graphs, path, st, info["iters"], round(time.time() - t, 3), flush=True)
'''

cases = [("c2", (64, 64, 128)), ("c3", (75, 150, 300)), ("c3", (150, 300, 600)), ("c3", (150, 300, 64))]
with open("/tmp/nccl_case.py", "w") as f:
    f.write(CASE)
for name, shape in cases:
    for graphs in (0, 1):
        for path in (1,):
            env = dict(os.environ, NCCL_DEBUG="WARN")
            t = time.time()
            r = subprocess.run([sys.executable, "/tmp/nccl_case.py", name, repr(shape), str(graphs), str(path), "40"],
                               capture_output=True, text=True, timeout=120, env=env)
            tail = (r.stdout + r.stderr).strip().splitlines()[-12:]
            print(f"== {name} {shape} graphs={graphs} path={path} rc={r.returncode} {time.time() - t:.1f}s", flush=True)
            for line in tail:
                print("   ", line[:200], flush=True)
