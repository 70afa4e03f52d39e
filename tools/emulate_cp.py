#!/usr/bin/env python
"""Row f1 measurement: DACP vs the paper's baseline plans on the attention path, one GPU.

    python tools/emulate_cp.py --config C5n8 [--schedulers skrull,dacp-only,rr,full-shard]

An N-rank CP group is emulated on ONE B200: every rank's packed micro-batch is run through the same
C-ABI kernels as production (RankStep phases; the all-gather / reduce-scatter replaced by device
copies), and each rank's attention calls (local / distributed, fwd / bwd) are timed with CUDA
events. The emulated step time is the Eq. 8-style sum over micro-batches of the slowest rank (P:184,
Eq. 1). Two figures per scheduler:
  * kernels only (no communication), and
  * with the exchange CHARGED as a stated LOWER bound: the bytes each rank must move over NVLink for
    the micro-batch -- all-gather receive (N-1) P Hkv d x 2 (K, V) x 2 B, reduce-scatter send
    (N-1) P Hkv d x 2 x 4 B (fp32) -- at the measured B200 peer-copy bandwidth of 770 GB/s per
    direction (B200_PROFILING.md; no latency, no collective overhead), composed per rank as Eq. 2
    executes it (R24 for the mirror): fwd = max(T_ag, T_local_fwd) + T_dist_fwd,
    bwd = T_dist_bwd + max(T_rs, T_local_bwd). A real collective only adds to this.
Schedulers:
  skrull     : GDS micro-batching (Alg. 2) + DACP (Alg. 1/3)
  dacp-only  : FIFO micro-batches under C*N tokens + DACP (the step-by-step ablation)
  rr         : FIFO micro-batches + round-robin placement (Alg. 4)
  full-shard : FIFO micro-batches, every sequence sharded (DeepSpeed-like baseline)
Prints one JSON line per scheduler.
"""
import argparse
import json

NVLINK_GBS = 770.0   # measured B200 peer copy, GB/s per direction (B200_PROFILING.md)
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def plans(sk, name, lens, C, N, h, hkv):
    """-> list of (mb_lens, mb_assign) for one global batch under scheduler `name`."""
    if name == "skrull":
        p = sk.skr_plan(lens, C, N, 1, h, hkv)
        out = []
        for j in range(int(p["n_mb_per_dp"][0])):
            idx = np.nonzero(p["mb_of_seq"] == j)[0]
            out.append((lens[idx], p["assign"][idx]))
        return out
    mbo, n = sk.skr_full_shard(lens, C, N)
    out = []
    for j in range(n):
        idx = np.nonzero(mbo == j)[0]
        ml = lens[idx]
        if name == "full-shard":
            a = np.full(len(ml), -1, np.int32)
        elif name == "dacp-only":
            a, _ = sk.skr_dacp(ml, C, N, h, hkv)
        elif name == "rr":
            a, _ = sk.skr_round_robin(ml, C, N)
        else:
            raise ValueError(name)
        out.append((ml, a))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5n8")
    ap.add_argument("--schedulers", default="skrull,dacp-only,rr,full-shard")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--weak", type=int, default=0,
                    help="C2 weak-scaled to N ranks exactly as bench.py --gpus N builds it (N x the batch, C=30720)")
    a = ap.parse_args()
    import torch
    from paper_2505_19609_b200 import skrull as sk
    from paper_2505_19609_b200.runtime import RankStep, loopback_step
    from synth import CONFIGS
    cfg = CONFIGS[a.config]
    lens = cfg.lengths(a.seed)
    N, C, shp = cfg.cp, cfg.bucket, cfg.shape
    if a.weak:
        cfg = CONFIGS["C2"]
        N, shp = a.weak, cfg.shape
        lens = np.concatenate([cfg.lengths(a.seed + r) for r in range(N)])
        C = cfg.bucket if N == 1 else 30720
        a.config = f"C2 weak x{N}"
    shape = sk.attn_shape(shp.hq, shp.hkv, shp.d, sk.SKR_BF16)
    useful = sum(14 * shp.d * shp.hq * int(S) * (int(S) + 1) // 2 for S in lens)
    g = torch.Generator(device="cuda").manual_seed(a.seed)
    for name in a.schedulers.split(","):
        mbs = plans(sk, name, lens, C, N, shp.hidden, shp.kv_hidden)
        step_ms, step_comm_ms, per_rank_tot, n_dist = 0.0, 0.0, np.zeros(N), 0
        comm_bytes = 0
        for ml, ma in mbs:
            n_dist += int((ma == -1).sum())
            ranks = [RankStep(shape, ml, ma, N, r) for r in range(N)]
            srcs = {k: [torch.randn(max(rs.rows, 1), shp.hq if k in ("q", "do") else shp.hkv, shp.d, device="cuda",
                                    generator=g).bfloat16() for rs in ranks] for k in ("q", "k", "v", "do")}
            loopback_step(ranks, srcs["q"], srcs["k"], srcs["v"], srcs["do"])      # warm-up
            kinds = ("fwd_local", "fwd_dist", "bwd_dist", "bwd_local")
            best = {k: np.full(N, np.inf) for k in kinds}
            for _ in range(a.reps):
                for rs in ranks:
                    rs.events = []
                loopback_step(ranks, srcs["q"], srcs["k"], srcs["v"], srcs["do"])
                torch.cuda.synchronize()
                for k in kinds:
                    t = np.array([sum(e0.elapsed_time(e1) for kk, e0, e1 in rs.events if kk == k) for rs in ranks])
                    best[k] = np.minimum(best[k], t)
            for rs in ranks:
                rs.events = None
            tot = sum(best[k] for k in kinds)
            # exchange lower bound of this micro-batch (zero without distributed sequences, R26)
            P = ranks[0].P if ranks[0].has_dist else 0
            ag = (N - 1) * P * shp.hkv * shp.d * 2 * 2
            rsb = (N - 1) * P * shp.hkv * shp.d * 2 * 4
            comm_bytes += ag + rsb
            t_ag, t_rs = ag / (NVLINK_GBS * 1e9) * 1e3, rsb / (NVLINK_GBS * 1e9) * 1e3
            with_comm = (np.maximum(t_ag, best["fwd_local"]) + best["fwd_dist"] + best["bwd_dist"]
                         + np.maximum(t_rs, best["bwd_local"]))
            step_ms += tot.max()
            step_comm_ms += with_comm.max()
            per_rank_tot += tot
            del ranks, srcs
            torch.cuda.empty_cache()
        out = {"scheduler": name, "config": a.config, "cp": N, "bucket": C, "micro_batches": len(mbs),
               "distributed_seqs": n_dist, "emulated_step_ms": step_ms,
               "useful_tflops_per_gpu": useful / (step_ms * 1e-3) / N / 1e12,
               "max_over_mean_rank_time": float(per_rank_tot.max() / per_rank_tot.mean()),
               "emulated_step_ms_with_comm_lb": step_comm_ms,
               "useful_tflops_per_gpu_with_comm_lb": useful / (step_comm_ms * 1e-3) / N / 1e12,
               "nvlink_bytes_per_rank": comm_bytes,
               "note": "attention kernels, one GPU, N ranks emulated; *_with_comm_lb adds the exchange at "
                       f"{NVLINK_GBS:.0f} GB/s per direction composed as Eq. 2 (a lower bound)"}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
