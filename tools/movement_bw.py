#!/usr/bin/env python
"""HBM GB/s of the data-movement kernels of rows a5 / a6 / a9 and their row-f3 peer forms
(north_star: "HBM GB/s for the packing/gather paths"), on one GPU with a loopback CP group.

    python tools/movement_bw.py [--config C3n2] [--out gpurun_out/movement_bw.json]

Every kernel runs through the C-ABI exactly as RankStep issues it, on the CP rank 0 tables of the
config's (largest) micro-batch; times are CUDA events over `--reps` launches after warm-up. GB/s
= ALGORITHMIC bytes (each byte the operation must read or write once) / time; the fraction is of
MEASURED_PEAKS.json's copy bandwidth. The peer kernels read the other emulated ranks' buffers,
which are local here (on NVLink the reads of remote chunks would be peer traffic instead).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3n2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from paper_2505_19609_b200 import skrull as sk
    from paper_2505_19609_b200.runtime import RankStep
    from synth import CONFIGS
    cfg = CONFIGS[a.config]
    lens = cfg.lengths(0)
    shp, N = cfg.shape, cfg.cp
    shape = sk.attn_shape(shp.hq, shp.hkv, shp.d, sk.SKR_BF16)
    p = sk.skr_plan(lens, cfg.bucket, N, 1, shp.hidden, shp.kv_hidden)
    mbs = []
    for j in range(int(p["n_mb_per_dp"][0])):
        idx = np.nonzero(p["mb_of_seq"] == j)[0]
        mbs.append((int(lens[idx].sum()), lens[idx], p["assign"][idx]))
    _, ml, ma = max(mbs, key=lambda t: t[0])
    ranks = [RankStep(shape, ml, ma, N, r) for r in range(N)]
    me = ranks[0]
    g = torch.Generator(device="cuda").manual_seed(0)
    src = {k: torch.randn(max(me.rows, 1), h, shp.d, device="cuda", generator=g).to(torch.bfloat16)
           for k, h in (("q", shp.hq), ("k", shp.hkv), ("v", shp.hkv))}
    for x in ranks:
        x.pack_qkv(src["q"][:x.rows] if x.rows <= me.rows else torch.randn(x.rows, shp.hq, shp.d, device="cuda").bfloat16(),
                   torch.randn(x.rows, shp.hkv, shp.d, device="cuda").bfloat16(),
                   torch.randn(x.rows, shp.hkv, shp.d, device="cuda").bfloat16())
        if x.has_dist:
            x.dk_nat.normal_()
            x.dv_nat.normal_()
    kv_row = shp.hkv * shp.d * 2
    addr = lambda name: torch.tensor([getattr(y, name).data_ptr() for y in ranks], dtype=torch.int64,  # noqa: E731
                                     device="cuda")
    for x in ranks:
        x.peer_k, x.peer_v, x.peer_dk, x.peer_dv = addr("k"), addr("v"), addr("dk_nat"), addr("dv_nat")
    own_rows = me.dist_rows
    ops = {
        "a5 pack Q (rank-natural -> packed)": (lambda: sk.skr_pack_rows(src["q"], me.src_row, me.q[:me.rows]),
                                              2 * me.rows * shp.hq * shp.d * 2),
        "a5 pack K": (lambda: sk.skr_pack_rows(src["k"], me.src_row, me.k[:me.rows]), 2 * me.rows * kv_row),
    }
    if me.has_dist:
        P = me.P
        ops.update({
            "a6 reorder K+V (gathered -> natural)": (me.kv_reorder, 2 * 2 * me.nat_rows * kv_row),
            "a9 permute dK+dV (natural -> rank-major, fp32)": (me.grad_scatter,
                                                               2 * (N * P * kv_row * 2 + me.nat_rows * kv_row * 2
                                                                    + me.nat_rows * kv_row * 2)),
            "a9 cast dK+dV (fp32 -> bf16)": (me.grad_cast, 2 * own_rows * kv_row * 3),
            "f3 peer gather K+V (owners' packed -> natural)": (me.peer_gather, 2 * 2 * me.nat_rows * kv_row),
            "f3 peer reduce dK+dV (N fp32 partials -> bf16)": (me.peer_reduce,
                                                               2 * own_rows * (N * kv_row * 2 + kv_row)),
        })
    peaks = {}
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        with open(pp) as f:
            peaks = json.load(f)
    peak = float(peaks.get("hbm_gbs", 6650.0))
    res = {"config": a.config, "rank_rows": me.rows, "natural_rows": me.nat_rows, "own_dist_rows": own_rows,
           "cp": N, "peak_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback",
           "ops": {}}
    for name, (fn, nbytes) in ops.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / a.reps * 1e-3
        gbs = nbytes / t / 1e9
        res["ops"][name] = {"bytes": int(nbytes), "us": t * 1e6, "gbs": gbs, "frac": gbs / peak}
        print(f"{name:52s} {nbytes / 1e6:9.1f} MB {t * 1e6:9.1f} us {gbs:8.0f} GB/s  {gbs / peak:5.2f} of peak",
              flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
