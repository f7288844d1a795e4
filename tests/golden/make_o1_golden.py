"""Write the dense O1 (truncated-SVD least squares) golden solution of a BASELINE config.

    python tests/golden/make_o1_golden.py c4          # ~10-13 min on 8 host cores

Calls only `oracle/` (dense.assemble_A, az.tsvd_lsq_multi) and the shared input generator; nothing
here comes from the CUDA path.  Stores the O1 coefficient vectors at the config's tol (the judge's
reference; "such solutions can be computed using a truncated SVD")
and at tol/100 (the oracle's own determinacy delta_det, reading F4(ii)), their relative residuals,
the truncation ranks and the leading singular values, as `tests/golden/<cfg>_o1.npz`.  The tests
evaluate the approximants from these coefficients with `oracle.az.evaluate` on the test grid.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2308_14490_b200 import inputs as I   # noqa: E402
from oracle import az as OA                      # noqa: E402
from oracle import dense as OD                   # noqa: E402


def main(name: str) -> None:
    cfg = I.get_config(name)
    t0 = time.time()
    A = OD.assemble_A(cfg)
    b = I.rhs(cfg)
    t1 = time.time()
    sols, s = OA.tsvd_lsq_multi(A, b, (cfg.tol, cfg.tol / 100.0))
    t2 = time.time()
    out = {"sigma_head": s[:16], "sigma_n": np.array(s.size), "assemble_s": np.array(t1 - t0),
           "svd_s": np.array(t2 - t1), "threads": np.array(os.cpu_count())}
    for tag, (x, k) in zip(("tol", "tol100"), sols):
        out[f"x_{tag}"] = x
        out[f"k_{tag}"] = np.array(k)
        out[f"res_{tag}"] = np.linalg.norm(A @ x - b, axis=0) / np.linalg.norm(b, axis=0)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}_o1.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: A {A.shape}, svd {t2 - t1:.1f} s, k {int(out['k_tol'])} / {int(out['k_tol100'])}, "
          f"res {out['res_tol']} / {out['res_tol100']} -> {path}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c4")
