#!/usr/bin/env python
"""Same-box context numbers (SURVEY §6 / BASELINE.md §2): library attention kernels on the SAME packed
local batch as this build's kernels, fwd and fwd+bwd, useful causal TFLOP/s (R32 convention:
4 / 10 * d * Hq per causal pair). Not the product path and not the bar -- context for the roofline:

  ours        skr_attn_fwd / skr_attn_bwd (this library, tcgen05), one local segment class
  fa2         flash_attn 2.8.3 flash_attn_varlen_func (the paper's kernel family, P:101, P:228;
              its wheel carries mma.sync code)
  fa4         vllm.vllm_flash_attn.cute flash_attn_varlen_func (FlashAttention-4, CuTe DSL, tcgen05)
  cudnn       torch SDPA with the cuDNN backend, one call per sequence (no varlen entry point),
              sequences >= --cudnn-min tokens only (reported on that subset)

    python tools/comparators.py [--config S4n1] [--reps 3]

Every library is optional: a failure prints {"impl": ..., "unavailable": "..."} and moves on.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(torch, fn, reps):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="S4n1")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--impls", default="ours,fa2,fa4,cudnn")
    ap.add_argument("--cudnn-min", type=int, default=4096)
    a = ap.parse_args()
    import torch
    from synth import CONFIGS
    cfg = CONFIGS[a.config]
    lens = [int(x) for x in cfg.lengths(0)]
    shp = cfg.shape
    T = sum(lens)
    pairs = sum(S * (S + 1) // 2 for S in lens)
    ff, fb = 4 * shp.d * shp.hq * pairs, 10 * shp.d * shp.hq * pairs
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda h: torch.randn(T, h, shp.d, device="cuda", generator=g).to(torch.bfloat16)  # noqa: E731
    q, k, v, do = mk(shp.hq), mk(shp.hkv), mk(shp.hkv), mk(shp.hq)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    mx = max(lens)
    base = {"config": a.config, "shape": f"Hq={shp.hq} Hkv={shp.hkv} d={shp.d}", "tokens": T, "seqs": len(lens)}

    def report(impl, t_f, t_fb, extra=None):
        out = dict(base, impl=impl, fwd_ms=t_f, fwd_tflops=ff / (t_f * 1e-3) / 1e12,
                   fwdbwd_ms=t_fb, fwdbwd_tflops=(ff + fb) / (t_fb * 1e-3) / 1e12)
        out.update(extra or {})
        print(json.dumps(out), flush=True)

    for impl in a.impls.split(","):
        try:
            if impl == "ours":
                from paper_2505_19609_b200 import skrull as sk
                from paper_2505_19609_b200.runtime import RankStep
                shape = sk.attn_shape(shp.hq, shp.hkv, shp.d, sk.SKR_BF16)
                rs = RankStep(shape, np.asarray(lens), np.zeros(len(lens), np.int32), 1, 0)
                rs.q[:T].copy_(q)
                rs.k[:T].copy_(k)
                rs.v[:T].copy_(v)
                rs.do[:T].copy_(do)
                t_f = timed(torch, rs.fwd_local, a.reps)
                t_b = timed(torch, rs.bwd_local, a.reps)
                report(impl, t_f, t_f + t_b)
                del rs
            elif impl == "fa2":
                from flash_attn import flash_attn_varlen_func as fa2
                qq, kk, vv = (x.clone().requires_grad_() for x in (q, k, v))
                f = lambda: fa2(qq, kk, vv, cu, cu, mx, mx, causal=True)  # noqa: E731
                t_f = timed(torch, f, a.reps)
                t_fb = timed(torch, lambda: f().backward(do), a.reps)
                report(impl, t_f, t_fb, {"version": __import__("flash_attn").__version__})
            elif impl == "fa4":
                from vllm.vllm_flash_attn.cute.interface import flash_attn_varlen_func as fa4
                qq, kk, vv = (x.clone().requires_grad_() for x in (q, k, v))
                f = lambda: fa4(qq, kk, vv, cu_seqlens_q=cu, cu_seqlens_k=cu, max_seqlen_q=mx,  # noqa: E731
                                max_seqlen_k=mx, causal=True)
                f1 = lambda: (lambda r: r[0] if isinstance(r, tuple) else r)(f())  # noqa: E731
                t_f = timed(torch, f1, a.reps)
                t_fb = timed(torch, lambda: f1().backward(do), a.reps)
                report(impl, t_f, t_fb)
            elif impl == "cudnn":
                import torch.nn.functional as F
                from torch.nn.attention import SDPBackend, sdpa_kernel
                sel = [(int(cu[i]), lens[i]) for i in range(len(lens)) if lens[i] >= a.cudnn_min]
                if not sel:
                    raise RuntimeError(f"no sequence >= {a.cudnn_min}")
                sp = sum(S * (S + 1) // 2 for _, S in sel)
                views = []
                for o, S in sel:
                    t = lambda x: x[o:o + S].transpose(0, 1)[None].detach().clone().requires_grad_()  # noqa: E731
                    views.append((t(q), t(k), t(v), do[o:o + S].transpose(0, 1)[None].contiguous()))

                def fwd(bwd=False):
                    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
                        for qq, kk, vv, dd in views:
                            y = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True, enable_gqa=True)
                            if bwd:
                                y.backward(dd)
                t_f = timed(torch, fwd, a.reps)
                t_fb = timed(torch, lambda: fwd(True), a.reps)
                f_sub, fb_sub = 4 * shp.d * shp.hq * sp, 14 * shp.d * shp.hq * sp
                print(json.dumps(dict(base, impl=impl, subset=f"{len(sel)} sequences >= {a.cudnn_min} tokens",
                                      fwd_ms=t_f, fwd_tflops=f_sub / (t_f * 1e-3) / 1e12, fwdbwd_ms=t_fb,
                                      fwdbwd_tflops=fb_sub / (t_fb * 1e-3) / 1e12,
                                      cudnn=torch.backends.cudnn.version())), flush=True)
        except Exception as e:  # noqa: BLE001 -- context numbers only
            print(json.dumps(dict(base, impl=impl, unavailable=f"{type(e).__name__}: {str(e)[:300]}")), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
