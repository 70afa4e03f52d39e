"""Debug timeline of one forward CTA (SKR_TRACE=1): per-KV-tile event times in cycles.

Needs an instrumented library: SKR_KERNEL_TRACE=1 python -m paper_2505_19609_b200.build --clean
(production builds compile the trace hooks out; rebuild without the variable afterwards)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKR_TRACE"] = "1"
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
ev = np.array([(x >> 48, x & ((1 << 48) - 1)) for x in buf[:n] if x])
ev = ev[np.argsort(ev[:, 1], kind="stable")]
t0 = ev[0, 1]
names = {1: "M S_A done", 2: "M S_B done", 3: "M PV_A done", 4: "M PV_B done", 5: "M S_A start", 6: "M S_B start", 7: "M PV_A start", 8: "M PV_B start", 10: "A s_full", 11: "A exps_done", 12: "A pv_done",
         13: "A p_arrive", 40: "T K issue", 41: "T V issue", 9: "M K ready, S busy", 20: "B s_full", 21: "B exps_done", 22: "B pv_done", 23: "B p_arrive"}
for e, t in ev[:260]:
    print(f"{t - t0:9d} {names.get(int(e), e)}")
