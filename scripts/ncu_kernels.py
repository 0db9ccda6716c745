"""One-GPU driver for ncu captures of the SM kernels: K1 (TMA bulk copy, local
256 MiB and sm_cap CTAs), K2 gather and K3 scatter at the config-4 shape
(32768 rows x 14336 B).  Used as:
    ncu --set full --clock-control none --import-source on -k regex:iccl_ -c 6 \
        -o gpurun_out/prof python scripts/ncu_kernels.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_00991_b200 import gather_rows, scatter_rows  # noqa: E402
from paper_2510_00991_b200._lib import lib  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
n = 256 << 20
a = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
b = torch.empty_like(a)
for ctas in (16, 148):
    assert lib.iccl_copy_sm(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), n, ctas, C.c_void_p(s.cuda_stream)) == 0
torch.cuda.synchronize()
assert torch.equal(a, b)
rows, H = 32768, 7168
tok = torch.randint(-32768, 32767, (4096, H), dtype=torch.int16, device="cuda").view(torch.bfloat16)
idx = torch.randint(0, 4096, (rows,), dtype=torch.int64, device="cuda")
g = gather_rows(tok, idx)
perm = torch.randperm(rows, device="cuda")
out = torch.empty_like(g)
scatter_rows(g, perm, out)
torch.cuda.synchronize()
print("ok")
