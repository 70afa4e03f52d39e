"""Microbenchmark: does an mbarrier probe after tcgen05.commit wait for the committed MMAs?

Groups of 2 / 4 / 8 SS UMMAs (128 x n x 16) issued warp-converged, each followed by a commit and then
(m=0) nothing, (m=1) a probe of an idle barrier, (m=2) a probe of the committed barrier,
(m=3) a plain shared load, (m=4) an idle-barrier probe with no commit. Cycles per group.
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
names = {0: "commit only", 1: "commit + idle probe", 2: "commit + own probe", 3: "commit + LDS", 4: "idle probe, no commit", 5: "in-block descriptors", 6: "one elected region"}
for gs_code, gs in ((2, 2), (0, 4), (1, 8)):
  for n in (64, 128):
    A = torch.randn(128, 128, device="cuda").bfloat16()
    B = torch.randn(n, 128, device="cuda").bfloat16()
    C = torch.zeros(128, n, device="cuda")
    cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
    for m in (range(7) if gs == 4 else range(5)):
        res = []
        for reps in (4, 68):
            sk._lib.skr_debug_umma_cycles(0, n, reps, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                          ctypes.c_void_p(C.data_ptr()), ctypes.c_void_p(cyc.data_ptr()),
                                          200 + 10 * gs_code + m)
            res.append(int(cyc[0].item()))
        extra = f"  own-group-complete {int(cyc[1].item())}/68" if m == 2 else ""
        print(f"gs={gs} n={n:3d} {names[m]:24s} cycles/group {(res[1] - res[0]) / 64:7.1f} (floor {gs * 128 * n / 256:.0f}){extra}")
