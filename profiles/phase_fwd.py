"""Per-warp phase accounting of the forward kernel (block (0, 0), the longest q tile).

Needs the phase-accounting build (no per-event traces, so the warps are not perturbed):
    SKR_KERNEL_TRACE=phase python -m paper_2505_19609_b200.build   # -> libskrull_trace.so
    python profiles/phase_fwd.py [d] [S]
Prints cycles per KV tile of every phase for warps 0-15 (softmax: head A 0-7, head B 8-15; warps
w and w+4 split the key columns of the same rows), the TMA warp (16) and the MMA thread (17).
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
S = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
hq, hkv = (14, 2) if d == 64 else (32, 8)
shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
q = torch.randn(S, hq, d, device="cuda").bfloat16(); k = torch.randn(S, hkv, d, device="cuda").bfloat16()
v = torch.randn_like(k); o = torch.zeros_like(q); lse = torch.zeros(hq, S, device="cuda")
fs = sk.make_segs(shape, [0, S], [0], [0], [S], "fwd")
buf = (ctypes.c_ulonglong * 8192)()
for _ in range(3):
    sk._lib.skr_debug_fwd_trace(buf, 8192)
    sk.skr_attn_fwd(shape, fs, q, k, v, o, lse)
    torch.cuda.synchronize()
sk._lib.skr_debug_fwd_trace(buf, 8192)
WG = int(os.environ.get("SKR_FWD_WG", "2"))   # softmax warpgroups per head of the build (kWG)
NW = 8 * WG + 2
a = np.array(buf[:NW * 8], dtype=np.int64).reshape(NW, 8)
n_kv = S // 128   # block (0, 0) runs the LPT-first (longest) q tile
names = {"sm": ["wait S", "ld S", "max+xchg", "wait PV", "store P", "-", "exps"] if WG == 2 else
         ["wait S", "ld S", "mask+max", "rescale O", "-", "-", "exps+st P"],
         NW - 2: ["wait slot", "issue"], NW - 1: ["wait K", "wait V", "wait S/P", "issue"]}
print(f"d={d} S={S}: cycles per KV tile (n_kv={n_kv})")
for w in range(NW):
    lab = names["sm"] if w < NW - 2 else names[w]
    row = "  ".join(f"{lab[i]} {a[w, i] / n_kv:7.0f}" for i in range(len(lab)))
    tot = a[w, :len(lab)].sum() / n_kv
    who = (f"{'A' if w < 4 * WG else 'B'}{(w // 4) % WG} w{w % 4}" if w < NW - 2 else
           ("TMA" if w == NW - 2 else "MMA"))
    print(f"{who:5s} total {tot:7.0f} | {row}")
