"""Timing probe of the vector operator on c3v: y = A x through maspcg_vv_apply, CUDA events, per variant
(MASPCG_VV_MARCH_DEBUG bit mask, see below; anything but 0 gives a wrong y;
MASPCG_VV_MARCH=0: the two-phase kernels).  Prints ms per apply."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_03398_b200 import inputs, maspcg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3v"
p = inputs.make_vv_problem(cfg)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
S = maspcg.Solver(p.nr, p.nt, p.np, p.rf, p.tf, p.pf)
S.vv_set_coefficients(T(p.nu), T(p.s))
S.vv_set_bc_r(p.wall_in, None, p.wall_out, None)
x = T(np.stack([inputs.white_noise(7 + c, p.nr, p.nt, 0, p.np) for c in range(3)], axis=1))
y = torch.empty_like(x)
# MASPCG_VV_MARCH_DEBUG bits: 1 no arithmetic, 2 no bulk copies, 4 no step waits, 8 no rows, 16 no terms,
# 32 return at entry
variants = [("full", {"MASPCG_VV_MARCH_DEBUG": "0"}), ("copies_only", {"MASPCG_VV_MARCH_DEBUG": "1"}),
            ("arith_only", {"MASPCG_VV_MARCH_DEBUG": "2"}), ("arith_nowait", {"MASPCG_VV_MARCH_DEBUG": "6"}),
            ("terms_only", {"MASPCG_VV_MARCH_DEBUG": "14"}), ("rows_only", {"MASPCG_VV_MARCH_DEBUG": "22"}),
            ("nothing", {"MASPCG_VV_MARCH_DEBUG": "7"}), ("return", {"MASPCG_VV_MARCH_DEBUG": "32"}),
             ("two_phase", {"MASPCG_VV_MARCH": "0"})]
for extra in sys.argv[2:]:
    k, v = extra.split("=")
    variants.append((extra, {k: v}))
for name, env in variants:
    old = {k: os.environ.get(k) for k in env}
    # the library honours the switch bits only with the 0x100 probe marker (vv_march.cu)
    os.environ.update({k: (str(int(v) | 0x100) if k == "MASPCG_VV_MARCH_DEBUG" and v != "0" else v)
                       for k, v in env.items()})
    for _ in range(3):
        S.vv_apply(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        S.vv_apply(x, y)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:14s} {e0.elapsed_time(e1) / n:8.3f} ms per apply", flush=True)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
S.close()
