"""The paper's eps regime: GPU solve vs O2 (same probes) and vs the exact f."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2308_14490_b200 import api, inputs as I
from oracle import az as OA
for fam, n, mb in [("interval_paper", 256, 4), ("interval_paper", 1024, 8), ("interval_paper", 4096, 8),
                   ("disk_paper", 32, 12), ("star_paper", 32, 12)]:
    cfg = I.make_config(fam, n)
    plan = api.Plan.from_config(cfg)
    b = I.rhs(cfg)
    theta = max(cfg.tol * 1e-2, 1e-12)
    x, rep = plan.solve(api.colmajor(torch.from_numpy(b).cuda()), theta, cfg.R, mb)
    x = x.cpu().numpy()
    g = I.test_grid(cfg)
    f = OA.evaluate(cfg, x, g)
    prob = OA.make_problem(cfg, "fft")
    r2 = OA.az_solve(prob, b, theta, cfg.R, cfg.seed, max_blocks=mb)
    f2 = OA.evaluate(cfg, r2.x.reshape(cfg.N, -1), g)
    sc = np.max(np.abs(g.exact))
    print(json.dumps({"cfg": cfg.name, "gpu_rank": rep["rank"], "gpu_probes": rep["probes"], "sat": rep["saturated"],
                      "o2_rank": r2.rank, "o2_probes": r2.probes_used, "err_gpu": float(np.max(np.abs(f - g.exact)) / sc),
                      "err_o2": float(np.max(np.abs(f2 - g.exact)) / sc), "gpu_vs_o2": float(np.max(np.abs(f - f2)) / sc),
                      "res_gpu": OA.relative_residual(prob, x, b).tolist(), "res_o2": OA.relative_residual(prob, r2.x.reshape(cfg.N, -1), b).tolist()}), flush=True)
