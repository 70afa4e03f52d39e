"""Microbenchmark: tensor-pipe cycles per 128 x n x 16 UMMA for each operand layout (one SM)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
names = {0: "SS A,B K-major", 1: "SS B MN-major", 2: "SS A,B MN-major", 3: "SS A thread-written", 4: "TS A in TMEM"}
for chains in (1, 2, 4):
  for n in (64, 128):
    for v in (0, 1, 4):
        A = torch.randn(128, 128, device="cuda").bfloat16()
        B = torch.randn(128, n, device="cuda").bfloat16() if v in (1, 2) else torch.randn(n, 128, device="cuda").bfloat16()
        C = torch.zeros(128, n, device="cuda")
        cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
        res = []
        for reps in (1, 64):
            sk._lib.skr_debug_umma_cycles(v, n, reps, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                          ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(cyc.data_ptr()), chains)
            res.append(int(cyc.item()))
        per = (res[1] - res[0]) / (63 * 8)
        print(f"chains={chains} n={n:3d} {names[v]:22s} cycles/UMMA {per:7.1f} (floor {128 * n / 256:.0f})")
