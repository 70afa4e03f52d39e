"""Microbenchmark: cycles per serialised group of g UMMAs (issue -> tcgen05.commit -> mbarrier wait)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
for n in (64, 128):
    for g in (1, 2, 4, 8, 16):
        A = torch.randn(128, 128, device="cuda").bfloat16(); B = torch.randn(n, 128, device="cuda").bfloat16()
        C = torch.zeros(128, n, device="cuda"); cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
        res = []
        for reps in (2, 66):
            sk._lib.skr_debug_umma_cycles(0, n, reps, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                          ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(cyc.data_ptr()), -g)
            res.append(int(cyc.item()))
        per = (res[1] - res[0]) / 64
        print(f"n={n:3d} group={g:2d}: {per:7.1f} cycles per group ({per / g:6.1f} per MMA; floor {128 * n / 256:.0f})")
