import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2308_14490_b200 import api, inputs as I
cfg = I.make_config("interval", 4096, nrhs=6, R=40)
plan = api.Plan.from_config(cfg)
b = I.rhs(cfg)
def sol(bb):
    x,_ = plan.solve(api.colmajor(torch.from_numpy(np.asfortranarray(bb)).cuda()), 1e-12, cfg.R, 1)
    return x.cpu().numpy()
x1 = sol(b); x3 = sol(-3*b); x2 = sol(2*b)
print("x(-3b)/x(b):", (x3/x1)[:3,0], "x(2b)/x(b):", (x2/x1)[:3,0])
x1b = sol(b); print("repeat b:", (x1b/x1)[:3,0])
