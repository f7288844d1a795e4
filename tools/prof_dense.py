"""Profiling driver for the wide dense kernels: blocked QR of an m x k matrix and the block-Jacobi
truncated SVD of a k x k triangular factor (random graded inputs).

    python tools/prof_dense.py qr m k | svd r nrhs
"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2308_14490_b200 import api
from paper_2308_14490_b200._lib import lib
mode = sys.argv[1]
g = torch.Generator(device="cuda").manual_seed(0)
if mode == "qr":
    m, k = int(sys.argv[2]), int(sys.argv[3])
    A = api.colmajor(torch.randn(m, k, dtype=torch.float64, device="cuda", generator=g))
    A2 = A.clone()
    api.qr_r(A2)
    torch.cuda.synchronize(); t = time.time()
    api.trace_enable(True)
    R = api.qr_r(A)
    torch.cuda.synchronize()
    dt = time.time() - t
    tr = api.trace_report()
    api.trace_enable(False)
    print(f"qr {m}x{k}: {dt*1e3:.1f} ms, {2*m*k*k/dt/1e12:.2f} TFLOP/s (2mk^2)")
    for name, (c, ms, u) in sorted(tr.items(), key=lambda kv: -kv[1][1]):
        extra = f" {u*1e-9/ms:.1f} TFLOP/s" if name in ("qrw_vtc", "qrw_upd") else ""
        print(f"  {name:12s} {c:5d} launches {ms:9.2f} ms{extra}")
else:
    r, nrhs = int(sys.argv[2]), int(sys.argv[3])
    X = torch.randn(2 * r, r, dtype=torch.float64, device="cuda", generator=g)
    X = X * torch.logspace(0, -11, r, dtype=torch.float64, device="cuda")[None, :]
    R = api.qr_r(api.colmajor(X))
    Rf = api.colmajor(torch.cat([R, torch.randn(r, nrhs, dtype=torch.float64, device="cuda", generator=g)], 1))
    torch.cuda.synchronize(); t = time.time()
    y, s, kk = api.tsvd_solve(Rf, r, nrhs, 1e-12)
    torch.cuda.synchronize()
    dt = time.time() - t
    print(f"svd r={r}: {dt*1e3:.1f} ms, rank {kk}, sweeps {lib().az_svd_sweeps_last(1)}, {13*8*r**3/dt/1e12:.2f} 'TFLOP/s' at 8r^3 x 13 sweeps")
