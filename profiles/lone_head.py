"""d = 64 forward: cost of the lone-head CTAs of odd GQA groups (Qwen2.5-0.5B: 7 q-heads per KV head).
Forward TFLOP/s of one local 32K sequence at hq = 14 / 16 / 12 with hkv = 2 (odd group: one lone head
per group; even groups: pairs only).

    python profiles/lone_head.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
from tools.calibrate import make_ranks, _time_fn, useful
S = 32768
for hq in (12, 14, 16):
    shape = sk.attn_shape(hq, 2, 64, sk.SKR_BF16)
    rs = make_ranks(torch, sk, shape, [S], [0], 1)[0][0]
    tf = min(_time_fn(torch, rs.fwd_local, reps=5) for _ in range(3))
    print(f"hq={hq} hkv=2 d=64 S={S}: fwd {tf * 1e3:7.3f} ms  {useful(S, hq, 64) * 4 / 14 / tf / 1e12:6.0f} TFLOP/s",
          flush=True)
    del rs
    torch.cuda.empty_cache()
