import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2308_14490_b200 import api, inputs as I
from paper_2308_14490_b200._lib import lib
cfg = I.get_config("c2")
plan = api.Plan.from_config(cfg)
b = api.colmajor(torch.from_numpy(I.rhs(cfg)).cuda())
S = api.empty_colmajor(plan.rows, cfg.R + cfg.nrhs)
plan.sketch(0, cfg.R, out=S[:, :cfg.R])
plan.apply_resid(b, out=S[:, cfg.R:])
R = api.qr_r(S)
Rn = R.cpu().numpy()
print("sv of R_S", np.linalg.svd(Rn[:64, :64], compute_uv=False)[[0, 19, 20, 21, 40, 63]])
for it in range(3):
    torch.cuda.synchronize(); t = time.time()
    y, sig, k = api.tsvd_solve(R, cfg.R, cfg.nrhs, 1e-12)
    torch.cuda.synchronize()
    print("rank", k, "ms", (time.time() - t) * 1e3, "sweeps", lib().az_debug_small_sweeps())
