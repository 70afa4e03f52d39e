"""Production forward kernel: cycles per (CTA, KV tile) on one causal sequence (no instrumentation).

    python profiles/fwd_period.py [S]

One sequence of S tokens, d=64 (Hq=14, Hkv=2) and d=128 (Hq=32, Hkv=8); the kernel is timed with
CUDA events and the time is converted to SM cycles per CTA tile iteration, assuming a balanced
grid: iterations = (#q tiles (t+1) summed) x head pairs / 148 SMs. Compare against the softmax
(MUFU) and MMA floors in DESIGN.md.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
clk = float(os.environ.get("SKR_SM_MHZ", "1965")) * 1e6
for d, hq, hkv in ((64, 14, 2), (128, 32, 8)):
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
    q = torch.randn(S, hq, d, device="cuda").bfloat16()
    k = torch.randn(S, hkv, d, device="cuda").bfloat16()
    v = torch.randn_like(k)
    o = torch.zeros_like(q)
    lse = torch.zeros(hq, S, device="cuda")
    fs = sk.make_segs(shape, [0, S], [0], [0], [S], "fwd")
    for _ in range(3):
        sk.skr_attn_fwd(shape, fs, q, k, v, o, lse)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        sk.skr_attn_fwd(shape, fs, q, k, v, o, lse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nt = S // 128
    iters = nt * (nt + 1) // 2 * (hq // 2) / 148
    flops = 4 * d * hq * S * (S + 1) / 2
    print(f"d={d:3d} S={S} fwd {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s  "
          f"{ms * 1e-3 * clk / iters:7.0f} cycles per CTA KV-tile (both heads)")
