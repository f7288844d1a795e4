import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2308_14490_b200 import api, inputs as I
cfg = I.get_config("c2")
plan = api.Plan.from_config(cfg)
b = I.rhs(cfg)
bh = torch.from_numpy(np.asfortranarray(b)).t().contiguous().pin_memory().t()
xh = [torch.empty((cfg.nrhs, cfg.N), dtype=torch.float64).pin_memory().t() for _ in range(2)]
for i in range(3):
    api.solve_host_pipelined(plan, bh, xh[i % 2], 1e-12, cfg.R, 1)
api.plan_sync(plan)
ts = []
t0 = time.time()
for i in range(6):
    t = time.time()
    api.solve_host_pipelined(plan, bh, xh[i % 2], 1e-12, cfg.R, 1)
    ts.append((time.time() - t) * 1e3)
t1 = time.time()
api.plan_sync(plan)
t2 = time.time()
print("per-call host ms:", [round(v, 2) for v in ts], "issue total", round((t1 - t0) * 1e3, 1), "sync", round((t2 - t1) * 1e3, 1))
