#!/usr/bin/env python
"""Row f2: on-box calibration of the cost model (App. C) and the Fig. 1b analog.

    python tools/calibrate.py [--out profiles/r01_calibration.json]            # one GPU
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/calibrate.py --comm-only

Measures on the B200 it runs on, through the C-ABI only (RankStep phases, skr_* calls):
  1. T_comp (Eq. 13): attention fwd + bwd kernel time of one local sequence of length S, for
     S = 256 ... 64K, per model shape; fitted with skr_fit_linear twice:
       against Eq. 12's FLOPs(S) (the paper's regressor, P:544 -- it also counts the 20bh^2 S linear
       terms this path does not run, so its fit is poor at short S), and
       against the useful causal attention FLOPs 14 d Hq S(S+1)/2 (R32, the work the kernels do).
  2. Fig. 1b analog: per-rank attention TFLOP/s of one sequence of length S sharded
     over a CP group of N ranks (zigzag chunks j and 2N-1-j, R20), every rank emulated on this GPU
     with the production kernels; the slowest rank sets the step.
  3. Memory(S): device bytes held by one rank's attention-path buffers for a micro-batch
     of S tokens (packed Q/K/V/O/dO/dQ/dK/dV, LSE, workspace), fitted linearly; the implied bucket
     size C = skr_bucket_size(budget) for the stated budget. This is the attention path only, not a
     whole model's activations (out of scope).
  4. T_comm (Eq. 15; Table 5 analog P:579-597): NCCL all-gather / reduce-scatter (the a6 / a9
     collectives, skr_comm) over 2 MB - 1 GB, max over ranks, fitted on >= 16 MB like S:563. Needs
     >= 2 GPUs (torchrun); on one GPU it is recorded as unavailable.
The JSON written here is read by tests/test_calibration.py, which compares the DACP heuristic
with the exhaustive optimum under the measured fits (the oracle is test infrastructure only).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"qwen05": (14, 2, 64), "qwen7": (28, 4, 128), "llama8": (32, 8, 128)}


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def time_rank(torch, steps, reps=5, warm=2):
    """Median over reps of the attention fwd + bwd C-ABI calls of every RankStep in `steps`
    (K/V for distributed chunks already in place), in seconds; per-rank list."""
    out = []
    for rs, src in steps:
        for _ in range(warm):
            _run_rank(rs, src)
        ts = []
        for _ in range(reps):
            a, b = _events(torch)
            a.record()
            _run_rank(rs, src)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        out.append(float(np.median(ts)))
    return out


def _time_fn(torch, fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = _events(torch)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def _run_rank(rs, src):
    if rs.loc_f.n_tiles:
        rs.fwd_local()
    if rs.has_dist:
        rs.fwd_dist()
        rs.bwd_dist()
    if rs.loc_b.n_tiles:
        rs.bwd_local()


def make_ranks(torch, sk, shape, lens, assign, N):
    """RankSteps of one micro-batch on this GPU, inputs packed, K/V exchanged by loopback copies."""
    from paper_2505_19609_b200.runtime import RankStep
    ranks, srcs = [], []
    g = torch.Generator(device="cuda").manual_seed(7)
    for r in range(N):
        rs = RankStep(shape, np.asarray(lens), np.asarray(assign, np.int32), N, r)
        R = max(rs.rows, 1)
        src = {k: torch.randn(R, h, shape.d, device="cuda", generator=g).to(torch.bfloat16)
               for k, h in (("q", shape.hq), ("k", shape.hkv), ("v", shape.hkv), ("do", shape.hq))}
        rs.pack_qkv(src["q"], src["k"], src["v"])
        rs.pack_do(src["do"])
        ranks.append(rs)
        srcs.append(src)
    if ranks[0].has_dist:
        P = ranks[0].P
        for x in ranks:
            for j, y in enumerate(ranks):
                ks, vs = y.kv_send()
                x.k_gath[j * P:(j + 1) * P].copy_(ks)
                x.v_gath[j * P:(j + 1) * P].copy_(vs)
            x.kv_reorder()
    # forward once so O / LSE exist for the backward
    for x in ranks:
        if x.loc_f.n_tiles:
            x.fwd_local()
        if x.has_dist:
            x.fwd_dist()
    torch.cuda.synchronize()
    return list(zip(ranks, srcs))


def useful(S, hq, d):
    return 14 * d * hq * S * (S + 1) // 2


def rank_useful(S, N, r, hq, d):
    tot = 0
    for c in (r, 2 * N - 1 - r):
        lo, hi = c * S // (2 * N), (c + 1) * S // (2 * N)
        tot += hi * (hi + 1) // 2 - lo * (lo + 1) // 2
    return 14 * d * hq * tot


def comp_sweep(torch, sk, lengths):
    res = {}
    for name, (hq, hkv, d) in SHAPES.items():
        shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
        rows = []
        for S in lengths:
            steps = make_ranks(torch, sk, shape, [S], [0], 1)
            t = time_rank(torch, steps)[0]
            rs = steps[0][0]
            tf = _time_fn(torch, rs.fwd_local)
            tb = _time_fn(torch, rs.bwd_local)
            rows.append({"S": S, "t_s": t, "fwd_s": tf, "bwd_s": tb, "eq12_flops": sk.skr_flops(S, hq * d, hkv * d),
                         "useful_flops": useful(S, hq, d), "tflops": useful(S, hq, d) / t / 1e12,
                         "fwd_tflops": useful(S, hq, d) * 4 / 14 / tf / 1e12,
                         "bwd_tflops": useful(S, hq, d) * 10 / 14 / tb / 1e12})
            del steps
            torch.cuda.empty_cache()
        x12 = [r["eq12_flops"] for r in rows]
        xu = [r["useful_flops"] for r in rows]
        y = [r["t_s"] for r in rows]
        a12, b12 = sk.skr_fit_linear(x12, y)
        au, bu = sk.skr_fit_linear(xu, y)

        def r2(x, a, b):
            yy = np.asarray(y)
            pred = a * np.asarray(x, np.float64) + b
            return float(1 - ((yy - pred) ** 2).sum() / ((yy - yy.mean()) ** 2).sum())
        res[name] = {"shape": {"hq": hq, "hkv": hkv, "d": d}, "points": rows,
                     "fit_eq12": {"slope_s_per_flop": a12, "intercept_s": b12, "r2": r2(x12, a12, b12)},
                     "fit_useful": {"slope_s_per_flop": au, "intercept_s": bu, "r2": r2(xu, au, bu),
                                    "tflops_asymptotic": 1e-12 / au if au > 0 else None}}
        print(f"[T_comp] {name}: " + " ".join(f"S={r['S']}:{r['tflops']:.0f} ({r['fwd_tflops']:.0f}/{r['bwd_tflops']:.0f})"
                                             for r in rows) + " TFLOP/s fwd+bwd (fwd/bwd)", flush=True)
    return res


def fig1b(torch, sk, lengths, degrees):
    hq, hkv, d = SHAPES["qwen7"]
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
    out = []
    for S in lengths:
        for N in degrees:
            if S < 2 * N:
                continue
            assign = [0] if N == 1 else [-1]
            steps = make_ranks(torch, sk, shape, [S], assign, N)
            ts = time_rank(torch, steps, reps=3)
            per = [rank_useful(S, N, r, hq, d) / t / 1e12 if N > 1 else useful(S, hq, d) / t / 1e12
                   for r, t in enumerate(ts)]
            step = max(ts)
            out.append({"S": S, "N": N, "rank_time_s": ts, "step_s": step,
                        "per_gpu_tflops": useful(S, hq, d) / step / N / 1e12, "rank_tflops": per})
            print(f"[fig1b] S={S} N={N}: per-GPU {out[-1]['per_gpu_tflops']:.0f} TFLOP/s "
                  f"(max/mean rank time {step / np.mean(ts):.3f})", flush=True)
            del steps
            torch.cuda.empty_cache()
    return {"shape": "qwen7 (28/4, d=128)", "points": out}


def mem_sweep(torch, sk, lengths, budget):
    from paper_2505_19609_b200.runtime import RankStep
    hq, hkv, d = SHAPES["qwen7"]
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
    pts = []
    for S in lengths:
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        base = torch.cuda.memory_allocated()
        rs = RankStep(shape, np.asarray([S]), np.asarray([0], np.int32), 1, 0)
        pts.append({"S": S, "bytes": int(torch.cuda.memory_allocated() - base)})
        del rs
    a, b = sk.skr_fit_linear([p["S"] for p in pts], [p["bytes"] for p in pts])
    C = sk.skr_bucket_size(budget, a, b)
    print(f"[memory] qwen7 attention path: {a:.0f} B/token + {b:.0f} B -> C = {C} tokens at {budget / 1e9:.0f} GB",
          flush=True)
    return {"shape": "qwen7 (28/4, d=128)", "points": pts, "fit": {"slope_bytes_per_token": a, "intercept_bytes": b},
            "budget_bytes": budget, "bucket_tokens": C}


def comm_sweep(torch, sk, sizes_mb):
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    comm = sk.Comm(world, rank)
    rows = []
    for mb in sizes_mb:
        n = mb * (1 << 20) // 2 // world                           # bf16 elements sent per rank (AG)
        send = torch.randn(n, device="cuda").to(torch.bfloat16)
        recv = torch.empty(n * world, device="cuda", dtype=torch.bfloat16)
        rs_send = torch.randn(n * world // 2, device="cuda")         # fp32, same bytes as the AG output
        rs_recv = torch.empty(n // 2, device="cuda")
        res = {}
        for kind in ("all_gather", "reduce_scatter"):
            fn = (lambda: comm.all_gather(send, recv)) if kind == "all_gather" else \
                 (lambda: comm.reduce_scatter_f32(rs_send, rs_recv))
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = _events(torch)
            a.record()
            for _ in range(10):
                fn()
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / 10 * 1e3], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[kind] = float(t.item())
        rows.append({"MB": mb, "all_gather_us": res["all_gather"], "reduce_scatter_us": res["reduce_scatter"]})
        if rank == 0:
            print(f"[T_comm] {mb} MB: AG {res['all_gather']:.1f} us, RS {res['reduce_scatter']:.1f} us", flush=True)
    comm.close()
    fits = {}
    for kind in ("all_gather", "reduce_scatter"):
        xs = [r["MB"] for r in rows if r["MB"] >= 16]
        ys = [r[f"{kind}_us"] for r in rows if r["MB"] >= 16]
        a, b = sk.skr_fit_linear(xs, ys)
        fits[kind] = {"slope_us_per_MB": a, "intercept_us": b}
    return {"world": world, "points": rows, "fit_ge16MB": fits}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_calibration.json"))
    ap.add_argument("--comm-only", action="store_true")
    ap.add_argument("--quick", action="store_true", help="fewer lengths (smoke of the tool)")
    a = ap.parse_args()
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    from paper_2505_19609_b200 import skrull as sk
    result = {"device": torch.cuda.get_device_name(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
        result["t_comm"] = comm_sweep(torch, sk, [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024])
        dist.destroy_process_group()
    else:
        result["t_comm"] = {"unavailable": "needs >= 2 GPUs (torchrun); gpurun boxes have one"}
    if not a.comm_only and rank == 0:
        lens = [256, 1024, 4096, 16384] if a.quick else [256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536]
        result["t_comp"] = comp_sweep(torch, sk, lens)
        result["fig1b"] = fig1b(torch, sk, [1024, 4096, 16384] if a.quick else [1024, 4096, 16384, 65536, 131072],
                                [1, 2, 4, 8])
        result["memory"] = mem_sweep(torch, sk, [4096, 16384, 65536], 64e9)
    if rank == 0:
        if a.comm_only and os.path.exists(a.out):
            with open(a.out) as f:
                old = json.load(f)
            old["t_comm"] = result["t_comm"]
            result = old
        with open(a.out, "w") as f:
            json.dump(result, f, indent=1)
        print(f"wrote {a.out}")


if __name__ == "__main__":
    main()
