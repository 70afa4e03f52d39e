"""Production backward kernel time on one causal sequence (d=64 Hq=14 Hkv=2, d=128 Hq=28 Hkv=4).

    python profiles/bwd_period.py [S]
Prints kernel-only time (preprocess + main + dQ convert, CUDA events) and useful TFLOP/s.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
S = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
for d, hq, hkv in ((64, 14, 2), (128, 28, 4)):
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
    q = torch.randn(S, hq, d, device="cuda").bfloat16(); k = torch.randn(S, hkv, d, device="cuda").bfloat16()
    v = torch.randn_like(k); do = torch.randn_like(q); o = torch.zeros_like(q); lse = torch.zeros(hq, S, device="cuda")
    fs = sk.make_segs(shape, [0, S], [0], [0], [S], "fwd"); bs = sk.make_segs(shape, [0, S], [0], [0], [S], "bwd")
    sk.skr_attn_fwd(shape, fs, q, k, v, o, lse)
    dq = torch.zeros_like(q); dk = torch.zeros_like(k); dv = torch.zeros_like(v)
    ws = torch.empty(sk.skr_attn_bwd_ws_bytes(shape, S) // 4 + 64, device="cuda")
    for _ in range(3):
        sk.skr_attn_bwd(shape, bs, q, k, v, o, do, lse, dq, dk, dv, 0, ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(10):
        sk.skr_attn_bwd(shape, bs, q, k, v, o, do, lse, dq, dk, dv, 0, ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    flops = 10 * d * hq * S * (S + 1) / 2
    print(f"d={d:3d} S={S} bwd {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s")
