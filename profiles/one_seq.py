"""One local sequence of length S through fwd + bwd (for ncu captures of a single launch).
    python profiles/one_seq.py [d] [S]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_19609_b200 import skrull as sk
from tools.calibrate import make_ranks
d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
hq, hkv = (28, 4) if d == 128 else (14, 2)
rs = make_ranks(torch, sk, sk.attn_shape(hq, hkv, d, sk.SKR_BF16), [S], [0], 1)[0][0]
rs.bwd_local()
torch.cuda.synchronize()
