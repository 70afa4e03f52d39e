"""Backward TFLOP/s of one local sequence vs its length (is the long-sequence slowdown the dQ
reduction traffic?). Run with the production library and with SKR_LIB_PATH=<variant>.

    python profiles/long_seq.py [d]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2505_19609_b200 import skrull as sk
from tools.calibrate import make_ranks, _time_fn, useful
d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
hq, hkv = (28, 4) if d == 128 else (14, 2)
shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
for S in (8192, 16384, 32768, 65536, 131072):
    rs = make_ranks(torch, sk, shape, [S], [0], 1)[0][0]
    tb = _time_fn(torch, rs.bwd_local, reps=3)
    tf = _time_fn(torch, rs.fwd_local, reps=3)
    print(f"d={d} S={S}: fwd {useful(S, hq, d) * 4 / 14 / tf / 1e12:6.0f}  bwd {useful(S, hq, d) * 10 / 14 / tb / 1e12:6.0f} TFLOP/s", flush=True)
    del rs
    torch.cuda.empty_cache()
