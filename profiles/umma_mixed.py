"""Microbenchmark: tensor-pipe cycles per UMMA for mixed MMA streams (one SM)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
names = {0: "SS/TS alternating, 1 acc", 1: "SS N=n / N=64 idesc alternating, 2 acc", 2: "SS, 2 acc alternating",
         3: "TS/SS alternating, 2 acc"}
for n in (64, 128):
    for m in range(4):
        A = torch.randn(128, 128, device="cuda").bfloat16(); B = torch.randn(n, 128, device="cuda").bfloat16()
        C = torch.zeros(128, n, device="cuda"); cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
        res = []
        for reps in (1, 64):
            sk._lib.skr_debug_umma_cycles(0, n, reps, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                          ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(cyc.data_ptr()), 100 + m)
            res.append(int(cyc.item()))
        print(f"n={n:3d} {names[m]:42s} {(res[1] - res[0]) / (63 * 8):7.1f} cycles/UMMA (floor {128 * n / 256:.0f})")
