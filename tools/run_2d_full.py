"""Full-size 2-D solves (BASELINE configs c3, c4, c5): time, probes, rank, per-kernel times, the
factorisation-reuse path (--factored).

    python tools/run_2d_full.py c4 [max_blocks]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_14490_b200 import api  # noqa: E402
from paper_2308_14490_b200 import inputs as I  # noqa: E402

name = sys.argv[1]
mb = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = I.get_config(name) if name in I.CONFIGS else I.make_config(name.split(':')[0], int(name.split(':')[1]))
t0 = time.time()
plan = api.Plan.from_config(cfg)
b = I.rhs(cfg)
bd = api.colmajor(torch.from_numpy(b).cuda())
theta = max(cfg.tol * 1e-2, 1e-12)
torch.cuda.synchronize()
t1 = time.time()
api.trace_enable(True)
x, rep = (None, {}) if "--fac-only" in sys.argv else plan.solve(bd, theta, cfg.R, mb)
torch.cuda.synchronize()
t2 = time.time()
tr = api.trace_report()
api.trace_enable(False)
x = x.cpu().numpy() if x is not None else None
rep = {k: v for k, v in rep.items() if k != "sigma"}
out = {"config": name, "plan_s": t1 - t0, "solve_s": t2 - t1, "report": rep,
       "kernels_ms": {k: round(v[1], 3) for k, v in sorted(tr.items(), key=lambda kv: -kv[1][1])[:14]}}
if "--factored" in sys.argv:
    torch.cuda.empty_cache()          # the solve's workspace goes back to the driver for the factor
    torch.cuda.synchronize(); t3 = time.time()
    fac = api.Factor(plan, theta, cfg.R, mb)
    torch.cuda.synchronize(); t4 = time.time()
    xf, _ = fac.solve(bd)
    torch.cuda.synchronize(); t5 = time.time()
    api.trace_enable(True)
    xf, frep = fac.solve(bd)
    torch.cuda.synchronize(); t6 = time.time()
    ftr = api.trace_report()
    api.trace_enable(False)
    # factored solves for several right-hand-side counts (the config's b tiled), CUDA-event timed
    sweep = {}
    for a in sys.argv:
        if a.startswith("--fac-nrhs="):
            for q in [int(v) for v in a.split("=")[1].split(",")]:
                bq = api.colmajor(bd[:, [j % bd.shape[1] for j in range(q)]].contiguous())
                fac.solve(bq)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                api.trace_enable(True)
                e0.record()
                for _ in range(3):
                    fac.solve(bq)
                e1.record(); torch.cuda.synchronize()
                qtr = api.trace_report()
                api.trace_enable(False)
                gbs = {k: round(v[2] / (v[1] / 1e3) / 1e9, 1) for k, v in qtr.items() if k.startswith("fac_") and v[1] > 0}
                sweep[q] = {"ms": e0.elapsed_time(e1) / 3, "GB/s": gbs,
                            "kernels_ms": {k: round(v[1] / 3, 3) for k, v in sorted(qtr.items(), key=lambda kv: -kv[1][1])[:4]}}
    out["factored"] = {"factorize_s": t4 - t3, "nrhs_sweep": sweep, "first_solve_s": t5 - t4, "solve_s": t6 - t5, "report": fac.report,
                       "solve_report": frep,
                       "kernels_ms": {k: round(v[1], 3) for k, v in sorted(ftr.items(), key=lambda kv: -kv[1][1])[:12]}}
# (accuracy against the manufactured solution and the oracle is checked by the test suite,
# tests/test_gpu_wide.py::test_solve_2d_full_size -- only tests/, smoke() and bench.py's CPU
# baseline run the oracle)
out["coef_norm_over_sqrtN"] = float(np.linalg.norm(x) / np.sqrt(cfg.N)) if x is not None else None
print(json.dumps(out))
