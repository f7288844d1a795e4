"""Per-launch timeline of one traced solve (diagnostics): start / end of every libaz launch in ms
from the solve's first launch, on whatever stream it ran, then the per-kernel totals.
    python tools/c2_timeline.py [config] [max_blocks]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["AZ_TRACE_TIMELINE"] = "1"

import torch  # noqa: E402

from paper_2308_14490_b200 import api  # noqa: E402
from paper_2308_14490_b200 import inputs as I  # noqa: E402

cfg = I.get_config(sys.argv[1] if len(sys.argv) > 1 else "c2")
plan = api.Plan.from_config(cfg)
b = api.colmajor(torch.from_numpy(I.rhs(cfg)).cuda())
theta = max(cfg.tol * 1e-2, 1e-12)
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for _ in range(1 if cfg.dim == 2 else 3):
    plan.solve(b, theta, cfg.R, mb)
torch.cuda.synchronize()
api.trace_enable(True)
plan.solve(b, theta, cfg.R, mb)
torch.cuda.synchronize()
for name, (cnt, ms, _) in sorted(api.trace_report().items(), key=lambda kv: -kv[1][1]):
    print(f"total {name:24s} {cnt:6d} {ms:10.3f} ms")
