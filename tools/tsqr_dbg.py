import os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2308_14490_b200 import api
from paper_2308_14490_b200._lib import lib
g = torch.Generator(device="cuda").manual_seed(0)
A = api.colmajor(torch.randn(1048577, 128, dtype=torch.float64, device="cuda", generator=g))
for it in range(2):
    B = A.clone()
    torch.cuda.synchronize()
    R = api.qr_r_partial(B, 64)
    torch.cuda.synchronize()
out = (ctypes.c_longlong * 3)()
lib().az_debug_tsqr(out)
print("CTA0 cycles: load", out[0], "panel", out[1], "update", out[2])
