"""Debug timeline of one forward CTA (SKR_TRACE=1): per-KV-tile event times in cycles.

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
hq, hkv = (14, 2) if d == 64 else (32, 8)
S = 8192
shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
q = torch.randn(S, hq, d, device="cuda").bfloat16(); k = torch.randn(S, hkv, d, device="cuda").bfloat16()
v = torch.randn_like(k); o = torch.zeros_like(q); lse = torch.zeros(hq, S, device="cuda")
fs = sk.make_segs(shape, [0, S], [0], [0], [S], "fwd")
buf = (ctypes.c_ulonglong * 8192)()
for _ in range(2):
    sk._lib.skr_debug_fwd_trace(buf, 8192)
    sk.skr_attn_fwd(shape, fs, q, k, v, o, lse)
    torch.cuda.synchronize()
n = sk._lib.skr_debug_fwd_trace(buf, 8192)
ev = np.array([(x >> 48, x & ((1 << 40) - 1), (x >> 40) & 0xFF) for x in buf[:n] if x])
ev = ev[np.argsort(ev[:, 1], kind="stable")]
t0 = ev[0, 1]
names = {1: "M S_A done", 2: "M S_B done", 3: "M PV_A done", 4: "M PV_B done", 5: "M S_A start", 6: "M S_B start", 7: "M PV_A start", 8: "M PV_B start", 10: "A s_full", 11: "A exps_done", 12: "A pv_done",
         13: "A p_arrive", 40: "T K issue", 41: "T V issue", 9: "M K ready, S busy", 60: "M PVA wait V", 61: "M PVB wait V", 62: "M PVA wait P", 63: "M PVB wait P", 64: "M S_A wait K", 65: "M S_B wait K", 66: "M S_A wait free", 67: "M S_B wait free", 30: "A w0 s_free", 31: "A w1 s_free", 32: "A w2 s_free", 33: "A w3 s_free", 34: "A w0 p_full", 35: "A w1 p_full", 36: "A w2 p_full", 37: "A w3 p_full", 50: "B w0 s_free", 51: "B w1 s_free", 52: "B w2 s_free", 53: "B w3 s_free", 54: "B w0 p_full", 55: "B w1 p_full", 56: "B w2 p_full", 57: "B w3 p_full", 20: "B s_full", 21: "B exps_done", 22: "B pv_done", 23: "B p_arrive"}
kinds = ["s_full", "s_free", "exps", "pv_done", "p_full"]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
print(f"{len(ev)} events")
for e, t, j in ev[lo:lo + 600]:
    e = int(e)
    if 30 <= e < 35 or 50 <= e < 55:   # per-warp softmax events: j | warp << 6
        name = f"{'A' if e < 50 else 'B'} w{j >> 6} {kinds[(e - 30) % 20]}"
        j = j & 63
    else:
        name = names.get(e, str(e))
    print(f"{t - t0:9d} {name:18s} j={j}")
