"""Block-Jacobi tuning probe: solve a config with different inner-sweep counts; print SVD time,
outer sweeps, rank and manufactured-solution error."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2308_14490_b200 import api, inputs as I
from paper_2308_14490_b200._lib import lib
from oracle import az as OA
name = sys.argv[1]
cfg = I.get_config(name) if name.startswith("c") else I.make_config(name.split("_")[0], int(name.split("_")[1]))
plan = api.Plan.from_config(cfg)
b = I.rhs(cfg)
bd = api.colmajor(torch.from_numpy(b).cuda())
grid = I.test_grid(cfg, 201)
for inner in [int(v) for v in sys.argv[2].split(",")]:
    lib().az_debug_jacobi(inner)
    x, rep = plan.solve(bd, 1e-12, cfg.R, 16)
    sw = lib().az_debug_jacobi(0)
    f = OA.evaluate(cfg, x.cpu().numpy(), grid)
    err = float(np.max(np.abs(f - grid.exact)) / np.max(np.abs(grid.exact)))
    print(json.dumps({"inner": inner, "outer_sweeps_last": sw, "ms_svd": rep["ms_svd"], "ms_qr": rep["ms_qr"],
                      "rank": rep["rank"], "probes": rep["probes"], "err": err}), flush=True)
