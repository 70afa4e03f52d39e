"""Microbenchmark: MUFU ex2 throughput on one SM (warp-instructions per cycle per SM sub-partition).

mode 0: pure ex2 chains; mode 1: each ex2 pair with FFMA2 + FADD2 + F2FP (the softmax instruction mix);
mode 2 / 3: packed ex2.approx.f16x2 / ex2.approx.ftz.bf16x2 (one instruction per element pair; the
printed rate counts ELEMENTS, two per instruction).
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
sink = torch.zeros(1, device="cuda")
for mode in (0, 1, 2, 3):
    for warps in (4, 8, 16):
        res = []
        for iters in (16, 272):
            sk._lib.skr_debug_mufu_cycles(warps, iters, mode, ctypes.c_void_p(cyc.data_ptr()), ctypes.c_void_p(sink.data_ptr()))
            res.append(int(cyc.item()))
        n_ex2 = (272 - 16) * 16 * warps * 32  # elements (modes 2/3: 8 instructions x 2 elements)
        c = res[1] - res[0]
        print(f"mode={mode} warps/SMSP={warps // 4}: {n_ex2 / c:5.1f} ex2/clk/SM  ({c / ((272 - 16) * 16 * warps / 4):5.2f} cycles per warp-ex2 per SMSP)")
