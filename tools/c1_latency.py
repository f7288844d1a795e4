"""c1 latency breakdown: per-kernel CUDA-event trace, stage times, Jacobi sweeps, host overhead.

    python tools/c1_latency.py [config] [max_blocks]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2308_14490_b200 import api, _lib  # noqa: E402
from paper_2308_14490_b200 import inputs as I  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = I.get_config(name)
plan = api.Plan.from_config(cfg)
b = api.colmajor(torch.from_numpy(I.rhs(cfg)).cuda())
x = api.empty_colmajor(plan.N, cfg.nrhs)
ws = torch.empty(plan.solve_workspace_bytes(cfg.nrhs, cfg.R, mb), dtype=torch.uint8, device="cuda")
theta = max(cfg.tol * 1e-2, 1e-12)
for _ in range(20):
    plan.solve(b, theta, cfg.R, mb, x=x, workspace=ws)
torch.cuda.synchronize()
K = 200
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    _, rep = plan.solve(b, theta, cfg.R, mb, x=x, workspace=ws)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / K * 1e3
print(f"{name} max_blocks {mb}: {e0.elapsed_time(e1) / K:.3f} ms/solve (events), {wall:.3f} ms wall, report {rep}")
print("jacobi sweeps", _lib.lib().az_svd_sweeps_last(0))
api.trace_enable(True)
plan.solve(b, theta, cfg.R, mb, x=x, workspace=ws)
torch.cuda.synchronize()
for k, v in sorted(api.trace_report().items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:28s} {v[0]:3d} launches {v[1] * 1e3:8.1f} us")
api.trace_enable(False)
