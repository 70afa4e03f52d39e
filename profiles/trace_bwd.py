"""Debug timeline of one backward CTA (SKR_TRACE=1): prints per-step event times in cycles.

Needs the instrumented library (production builds compile the trace hooks out):
    SKR_KERNEL_TRACE=1 python -m paper_2505_19609_b200.build   # -> libskrull_trace.so (loaded below)"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKR_TRACE"] = "1"
os.environ.setdefault("SKR_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                   "paper_2505_19609_b200", "libskrull_trace.so"))
import torch
from paper_2505_19609_b200 import skrull as sk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
hq, hkv = (14, 2) if d == 64 else (28, 4)
S = 8192
shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
q = torch.randn(S, hq, d, device="cuda").bfloat16(); k = torch.randn(S, hkv, d, device="cuda").bfloat16()
v = torch.randn_like(k); do = torch.randn_like(q)
o = torch.zeros_like(q); lse = torch.zeros(hq, S, device="cuda")
fs = sk.make_segs(shape, [0, S], [0], [0], [S], "fwd"); bs = sk.make_segs(shape, [0, S], [0], [0], [S], "bwd")
sk.skr_attn_fwd(shape, fs, q, k, v, o, lse)
dq = torch.zeros_like(q); dk = torch.zeros_like(k); dv = torch.zeros_like(v)
ws = torch.empty(sk.skr_attn_bwd_ws_bytes(shape, S) // 4 + 64, device="cuda")
for _ in range(2):
    buf = (ctypes.c_ulonglong * 8192)()
    sk._lib.skr_debug_bwd_trace(buf, 8192)
    sk.skr_attn_bwd(shape, bs, q, k, v, o, do, lse, dq, dk, dv, 0, ws)
    torch.cuda.synchronize()
n = sk._lib.skr_debug_bwd_trace(buf, 8192)
ev = np.array([(x >> 48, x & ((1 << 48) - 1)) for x in buf[:n] if x])
ev = ev[np.argsort(ev[:, 1], kind="stable")]
t0 = ev[0, 1]
names = {1: "M s_free", 2: "M qdo", 3: "M p_full", 4: "M ds_full", 5: "M dq_empty", 10: "C s_full", 11: "C p_arrive",
         12: "C dp_full", 13: "C ds_arrive", 14: "C qdo_full", 20: "Q dq_full", 21: "Q dq_empty_arr"}
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0          # optional window start (cycles after t0)
sel = [(e, t) for e, t in ev if t - t0 >= lo][:200]
for e, t in sel:
    print(f"{t - t0:9d} {names.get(int(e), e)}")
