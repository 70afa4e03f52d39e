"""Per-warp phase accounting of the backward kernel (block (0, 0), the LPT-first KV tile).

    SKR_KERNEL_TRACE=phase python -m paper_2505_19609_b200.build   # -> libskrull_trace.so
    python profiles/phase_bwd.py [d] [S]
Cycles per step (one query tile of one head against the CTA's KV tile) of every phase: compute
warpgroups (warps 0-7), dQ warpgroup (8-11), MMA thread (13).
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKR_TRACE"] = "1"
os.environ.setdefault("SKR_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                   "paper_2505_19609_b200", "libskrull_trace.so"))
import numpy as np
import torch
from paper_2505_19609_b200 import skrull as sk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
hq, hkv = (14, 2) if d == 64 else (28, 4)
shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
q = torch.randn(S, hq, d, device="cuda").bfloat16(); k = torch.randn(S, hkv, d, device="cuda").bfloat16()
v = torch.randn_like(k); do = torch.randn_like(q)
o = torch.zeros_like(q); lse = torch.zeros(hq, S, device="cuda")
fs = sk.make_segs(shape, [0, S], [0], [0], [S], "fwd"); bs = sk.make_segs(shape, [0, S], [0], [0], [S], "bwd")
sk.skr_attn_fwd(shape, fs, q, k, v, o, lse)
dq = torch.zeros_like(q); dk = torch.zeros_like(k); dv = torch.zeros_like(v)
ws = torch.empty(sk.skr_attn_bwd_ws_bytes(shape, S) // 4 + 64, device="cuda")
buf = (ctypes.c_ulonglong * 8192)()
for _ in range(3):
    sk._lib.skr_debug_bwd_trace(buf, 8192)
    sk.skr_attn_bwd(shape, bs, q, k, v, o, do, lse, dq, dk, dv, 0, ws)
    torch.cuda.synchronize()
sk._lib.skr_debug_bwd_trace(buf, 8192)
a = np.array(buf[:112], dtype=np.int64).reshape(14, 8)
n = int(a[13, 7])
comp = ["wait S", "ld S", "exp", "wait dV", "st P", "wait dP", "dS math", "st dS"]
dqn = ["wait dQ", "wait tile", "TMEM>smem", "reduce"]
mma = ["s_free", "qdo", "p_full", "dp_free", "ds_full", "dq_empty", "issue"]
print(f"d={d} S={S}: cycles per step (n_steps={n})")
for w in list(range(8)) + list(range(8, 12)) + [13]:
    lab = comp if w < 8 else dqn if w < 12 else mma
    row = "  ".join(f"{lab[i]} {a[w, i] / n:6.0f}" for i in range(len(lab)))
    print(f"w{w:<3d} total {a[w, :len(lab)].sum() / n:6.0f} | {row}")
