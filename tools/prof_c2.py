"""Profiling driver (ncu): one c2 solve ("solve") or the sketch + QR + SVD parts once ("parts").

    python tools/prof_c2.py [solve|parts] [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2308_14490_b200 import api  # noqa: E402
from paper_2308_14490_b200 import inputs as I  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "solve"
cfg = I.get_config(sys.argv[2] if len(sys.argv) > 2 else "c2")
plan = api.Plan.from_config(cfg)
b = api.colmajor(torch.from_numpy(I.rhs(cfg)).cuda())
theta = max(cfg.tol * 1e-2, 1e-12)
if mode == "solve":
    x, rep = plan.solve(b, theta, cfg.R, 1)
    torch.cuda.synchronize()
    print(rep)
else:
    S = api.empty_colmajor(plan.rows, cfg.R + cfg.nrhs)
    plan.sketch(0, cfg.R, out=S[:, :cfg.R])
    plan.apply_resid(b, out=S[:, cfg.R:])
    R = api.qr_r(S)
    y, sig, k = api.tsvd_solve(R, cfg.R, cfg.nrhs, theta)
    torch.cuda.synchronize()
    print("rank", k)
