#!/usr/bin/env python
"""Bench: DACP/GDS-scheduled packed varlen causal attention fwd+bwd on B200 (the Skrull hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config NAME]

One step = one pass of the whole hot path over one global batch: for
every GDS micro-batch of this rank, pack Q/K/V (a5), K/V all-gather + reorder for distributed
sequences (a6, N>1), attention forward local-then-distributed (a7), pack dO, attention backward
distributed-then-local (a8), dK/dV reduce-scatter + cast (a9, N>1). The host plan (a1-a4, the
paper's "near-zero overhead" DataLoader step) is computed once per global batch before the
timed region and reported as `plan_us`.

Metric (BASELINE.json): useful causal attention TFLOP/s fwd+bwd = sum_seq 14*d*Hq*S(S+1)/2 (R32)
divided by the step time (max over ranks), whole-job aggregate. Inputs (Q, K, V, dO of the batch
plus activations) exceed the 126 MB L2, so no explicit flush is done between steps.

Workload (the same at every N, so BENCH and SCALE share it): S4n{N} -- BASELINE configs[3]'s
global batch (Qwen2.5-7B attention shape 28/4, d=128; 511 `short1k` sequences + one 128K) with
the SURVEY §8(d) strong-scaling BucketSize of that CP degree (512K / 96K / 48K / 24K tokens per
rank at N = 1 / 2 / 4 / 8, so DACP shards the 128K sequence for N >= 2 and the plan floor stays
<= 1.001). `--config NAME` selects another (C2 = configs[1] weak-scaled by N; C5n*/C5Hn* =
configs[4]; C3n*, C4).

Rank 0 prints ONE JSON line. Under torchrun (N>1) the ranks form a DP x CP grid (--dp, default 1:
one CP group of N ranks; row f4): CP groups are blocks of N/dp consecutive ranks, GDS/LPT bins the
batch over the DP ranks and DACP places inside each CP group.

Timing: W untimed steps; then K steps between a barrier + synchronize on
both sides. Before every step the ranks align their device timelines with a 1-element all-reduce
on the main stream, and each step is bracketed by CUDA events; the library records 8 more events
around its attention calls inside each composite step (skr_cp_step.timing_events), so the
dominant kernel's time for the roofline comes from the SAME timed pass as the headline. Reported:
the whole-loop time (max over ranks) as `ms_per_step`, the per-step max over ranks / mean over
ranks with median and p10-p90, and the part of the step outside the attention calls.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS  # noqa: E402
from synth.configs import Shape  # noqa: E402

METRIC = "useful causal attn TFLOP/s fwd+bwd"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="workload (default: S4n{N}, strong-scaled over the CP group)")
    ap.add_argument("--dp", type=int, default=1, help="DP degree of the DP x CP grid (CP = N / dp)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer", "peer1", "ring"],
                    help="CP exchange: NCCL all-gather / reduce-scatter; 'peer': row f3 step two (peer gather, "
                         "dK/dV reduced from the backward kernel's epilogue into the owners' memory); 'peer1': "
                         "row f3 step one (peer gather + peer-reduce pass); 'ring': row f4's alternative, ring CP "
                         "(K/V hop around the CP group point-to-point, partial attentions merged)")
    ap.add_argument("--bwd-band", type=int, default=None,
                    help="query-band height of the backward work items (skr_tiles_bwd; default: the library's)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


# ----------------------------------------------------------------------------- workload
DEFAULT_WORKLOAD = "S4"   # S4n{cp}: configs[3]'s batch, strong-scaled over the CP group


def workload(args, world):
    """Global batch lengths, shape, CP degree and BucketSize for this run:
    -> (name, cfg, lens, shape, cp, bucket, scaling). cp = world // dp (DP x CP grid)."""
    dp = args.dp
    if dp < 1 or world % dp:
        raise SystemExit(f"--dp {dp} does not divide {world} ranks")
    cp = world // dp
    name = args.config or f"{DEFAULT_WORKLOAD}n{cp}"
    if name == "C2":
        cfg = CONFIGS[name]
        # weak scaling of configs[1]: N x (63 long-tail + one 32K) sequences over the DP x CP grid.
        # With CP >= 2 the BucketSize is set below the longest sequence (R33) so DACP shards it:
        # 30720 gives 3 micro-batches per rank with only the 32K sequences sharded at N = 8 and plan
        # floors 1.006 / 1.070 / 1.088 at N = 2 / 4 / 8 (24576: 4 / 4 / 3 micro-batches, 19 sequences
        # sharded at N = 8, floors 1.008 / 1.074 / 1.088).
        lens = np.concatenate([cfg.lengths(args.seed + r) for r in range(world)])
        bucket = cfg.bucket if cp == 1 else 30720
        return name, cfg, np.asarray(lens, np.int64), cfg.shape, cp, bucket, "weak"
    if name not in CONFIGS:
        raise SystemExit(f"unknown config {name}; one of {sorted(CONFIGS)}")
    cfg = CONFIGS[name]
    if cfg.cp != cp:
        raise SystemExit(f"config {name} is for CP={cfg.cp}; {world} ranks with --dp {dp} give CP={cp}")
    scaling = "strong" if name.startswith("S4") else "weak"
    return name, cfg, np.asarray(cfg.lengths(args.seed), np.int64), cfg.shape, cp, cfg.bucket, scaling


def useful_flops(lens, shape: Shape, part="fwdbwd"):
    pairs = sum(int(S) * (int(S) + 1) // 2 for S in lens)
    per = {"fwd": 4, "bwd": 10, "fwdbwd": 14}[part]
    return per * shape.d * shape.hq * pairs


def rank_pairs(mb_lens, assign, cp, rank):
    tot = 0
    for S, a in zip(mb_lens, assign):
        S = int(S)
        if a == rank:
            tot += S * (S + 1) // 2
        elif a == -1:
            for c in (rank, 2 * cp - 1 - rank):
                lo, hi = c * S // (2 * cp), (c + 1) * S // (2 * cp)
                tot += hi * (hi + 1) // 2 - lo * (lo + 1) // 2
    return tot


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap,power.limit"

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        def num(i):
            v = []
            for r in self.rows:
                try:
                    v.append(float(r[i]))
                except (IndexError, ValueError):
                    pass
            return v
        pw, pl = num(2), num(8)
        # clocks and power limit beside the numbers
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": float(np.median(pw)) if pw else None, "power_limit_w": max(pl) if pl else None}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def ncu_traffic(workload, world, kind):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed `ncu --set full`
    capture summary (profiles/ncu_summary.json, written by profiles/summarize_ncu.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            j = json.load(f)
        e = j[f"{workload}/n{world}"][f"attn_{kind}"]
        return float(e["dram_bytes"]), e.get("source", "profiles/ncu_summary.json")
    except Exception:
        return None


def eval_prediction(sk, all_mbs, cp, bucket, shp):
    """Row f2: the paper's evaluator (Eq. 8 = max over DP ranks of the sum over micro-batches of
    Eq. 1's TDACP, skr_eval_tdacp) with the B200 T_comp fit of profiles/r01_calibration.json (against
    Eq. 12's FLOPs, as the paper fits it) and Table 5's all-gather fit for T_comm (no
    NVLink sweep yet), in ms -- printed next to the measured step. None without a calibration."""
    names = {(14, 2, 64): "qwen05", (28, 4, 128): "qwen7", (32, 8, 128): "llama8"}
    path = os.path.join(ROOT, "profiles", "r01_calibration.json")
    name = names.get((shp.hq, shp.hkv, shp.d))
    if not name or not os.path.exists(path):
        return None
    with open(path) as f:
        fit = json.load(f)["t_comp"][name]["fit_eq12"]
    comp = (fit["slope_s_per_flop"], fit["intercept_s"])
    comm = (6.256e-6 / (1 << 20), 116.5e-6)          # Table 5 all_gather, per byte (R25: 2 B/elem)
    worst = 0.0
    for d_mbs in all_mbs:
        t = 0.0
        for ml, ma in d_mbs:
            r = sk.skr_eval_tdacp(ml, ma, bucket, cp, shp.hidden, shp.kv_hidden, comp, comm, bytes_per_elem=2.0)
            t += r["tdacp"]
        worst = max(worst, t)
    return worst * 1e3


# ----------------------------------------------------------------------------- CPU oracle leg
def cpu_oracle_sample(lens, shape: Shape, seconds: float, seed: int = 0):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload: sequences taken
    shortest-first while the projected time (measured FLOP rate so far x the next sequence's useful
    FLOPs) stays within `seconds`. Returns (TFLOP/s, n_seqs, tokens, wall_s, useful_flops)."""
    from oracle.attention import attn_bwd, attn_fwd
    from synth import seq_tensors
    order = np.argsort(lens, kind="stable")
    done_flops, n, toks, t_used = 0, 0, 0, 0.0
    for k in order:
        S = int(lens[k])
        f = useful_flops([S], shape)
        if n > 0 and t_used + f / (done_flops / t_used) > seconds:
            break
        x = seq_tensors(seed, int(k), S, shape.hq, shape.hkv, shape.d)
        t0 = time.perf_counter()
        attn_fwd(x["q"], x["k"], x["v"])
        attn_bwd(x["q"], x["k"], x["v"], x["do"])
        t_used += time.perf_counter() - t0
        done_flops += f
        n += 1
        toks += S
    return done_flops / t_used / 1e12, n, toks, t_used, done_flops


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    name, cfg, lens, shape, cp, bucket, scaling = workload(args, world)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    tot_flops, tot_t = 0, 0.0
    sample = None
    for i in range(args.warmup + args.steps):
        v, n, toks, t, f = cpu_oracle_sample(lens, shape, per_step, args.seed)
        if i >= args.warmup:
            # the sample size is time-budgeted and may differ between iterations: sum the work
            # and the time over the timed iterations (not the last iteration's work / mean time)
            tot_flops += f
            tot_t += t
            sample = f"{n} shortest sequences of the batch ({toks} tokens), fp64 naive attention fwd+bwd"
    value = tot_flops / tot_t / 1e12
    cores = len(os.sched_getaffinity(0))
    out = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
           "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": name, "shape": f"Hq={shape.hq} Hkv={shape.hkv} d={shape.d}", "cp": cp,
                      "bucket": int(bucket), "global_batch": int(len(lens))},
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
def pick_peak(peaks, clocks, timed_s):
    """Roofline denominator: the measured BURST bf16 GEMM rate, unless the timed region ran for
    seconds at power-capped clocks (median SM clock under load < 90 % of max), where the SUSTAINED
    figure of the same measurement applies (B200_PROFILING.md)."""
    burst = float(peaks.get("bf16_tflops", 1590.0))
    sus = float(peaks.get("bf16_tflops_sustained", burst))
    mhz, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    sustained = bool(timed_s >= 2.0 and mhz and mx and mhz < 0.9 * mx)
    return (sus, "bf16_tflops_sustained") if sustained else (burst, "bf16_tflops"), burst, sus


def pctl(x, q):
    return float(np.percentile(np.asarray(x, np.float64), q))


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # SKR_BENCH_BACKEND=gloo: control plane over gloo with every rank on the visible GPUs modulo
    # their count -- a functional multi-rank run on ONE GPU for --exchange peer (timings meaningless)
    backend = os.environ.get("SKR_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2505_19609_b200 import skrull as sk
    from paper_2505_19609_b200.runtime import BufferPool, RankStep, dp_micro_batches, grid_coords

    dp = args.dp
    name, cfg, lens, shp, cp, bucket, scaling = workload(args, world)
    dp_rank, cp_rank, _ = grid_coords(rank, world, dp)
    shape = sk.attn_shape(shp.hq, shp.hkv, shp.d, sk.SKR_BF16)
    h, hkv = shp.hidden, shp.kv_hidden

    # ---- a1-a4: host plan (every rank computes the identical plan); the Python scheduler
    # oracle is timed beside it on rank 0 (the paper's "near-zero overhead")
    t0 = time.perf_counter()
    plan = sk.skr_plan(lens, bucket, cp, dp, h, hkv)
    plan_us = (time.perf_counter() - t0) * 1e6
    all_mbs = [[(ml, ma) for _, ml, ma in dp_micro_batches(plan, lens, d)] for d in range(dp)]
    mbs = all_mbs[dp_rank]
    n_mb = len(mbs)

    comm = None
    if cp > 1:
        # one communicator per CP group (every rank takes part in creating every group)
        groups = [dist.new_group(list(range(d * cp, (d + 1) * cp))) for d in range(dp)]
        if args.exchange in ("peer", "peer1"):
            comm = sk.PeerComm(cp, cp_rank, group=groups[dp_rank])
        else:
            comm = sk.Comm(cp, cp_rank, group=groups[dp_rank], src=dp_rank * cp)
    nccl_comm = comm if (comm is not None and args.exchange in ("nccl", "ring")) else None
    ring = args.exchange == "ring" and comm is not None   # row f4: ring CP (NCCL point-to-point hops)
    side = torch.cuda.Stream(priority=-1)
    main = torch.cuda.current_stream()
    steps = []
    g = torch.Generator(device="cuda")
    # the micro-batches run one after another: their working buffers come from one shared pool
    pool = BufferPool()
    rsteps = [RankStep(shape, ml, ma, cp, cp_rank, alloc=pool.reserve, band_rows=args.bwd_band, ring=ring)
              for ml, ma in mbs]
    pool.materialize()
    for rs in rsteps:
        rs.rebind(pool.get)
    for j, rs in enumerate(rsteps):
        if args.exchange in ("peer", "peer1") and comm is not None:
            rs.connect_peer(comm)              # collective inside the CP group
        g.manual_seed(args.seed * 1_000_003 + rank * 1009 + j)
        R = max(rs.rows, 1)
        src = {k: torch.randn(R, hh, shp.d, device="cuda", generator=g).to(torch.bfloat16)
               for k, hh in (("q", shp.hq), ("k", shp.hkv), ("v", shp.hkv), ("do", shp.hq))}
        steps.append((rs, src))

    def fwd_bwd(rs, src, ev_do=None, timing=None):
        # ev_do (e2e only): the backward waits for this micro-batch's dO copy, the forward does not
        if ring:
            rs.forward_ring(src["q"], src["k"], src["v"], comm, side)
            if ev_do is not None:
                torch.cuda.current_stream().wait_event(ev_do)
            rs.backward_ring(src["do"], comm, side)
        elif args.exchange in ("peer", "peer1") and comm is not None:
            rs.forward_peer(src["q"], src["k"], src["v"], side)
            if ev_do is not None:
                torch.cuda.current_stream().wait_event(ev_do)
            (rs.backward_peer_fused if args.exchange == "peer" else rs.backward_peer)(src["do"], side)
        else:
            rs.forward(src["q"], src["k"], src["v"], comm, side, timing=timing)
            if ev_do is not None:
                torch.cuda.current_stream().wait_event(ev_do)
            rs.backward(src["do"], comm, side, timing=timing)

    def one_step(timing=None):
        for j, (rs, src) in enumerate(steps):
            fwd_bwd(rs, src, timing=timing[j] if timing is not None else None)

    align_buf = torch.zeros(1, device="cuda")

    def align():
        # per-step alignment of the ranks' device timelines
        if world > 1:
            if backend == "nccl":
                dist.all_reduce(align_buf)
            else:
                torch.cuda.synchronize()
                dist.barrier()

    def sync():
        # comm-aware synchronize: an NCCL error or a dead peer surfaces as an exception after the
        # timeout instead of a hang (skr_comm_wait polls ncclCommGetAsyncError); the peer exchange's
        # timed-out waits are reported by PeerComm.check
        if nccl_comm is not None:
            nccl_comm.wait(main, timeout_s=600.0)
        torch.cuda.synchronize()
        if comm is not None and args.exchange in ("peer", "peer1"):
            comm.check()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(args.warmup, 0)):
        one_step()
    sync()
    barrier()

    # per-(step, micro-batch) attention timing events (recorded by the library inside the composite
    # steps); created up front so recording them costs nothing in the loop
    K = args.steps
    use_lib_timing = not (args.exchange in ("peer", "peer1", "ring") and comm is not None)
    timing = None
    if use_lib_timing:
        timing = [[[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(n_mb)] for _ in range(K)]
        for per_step in timing:
            for evs in per_step:
                for e in evs:
                    e.record(main)
    else:
        for rs, _ in steps:
            rs.events = []                     # the peer path's per-call events (fwd / bwd kinds)
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    sync()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sync()
    barrier()
    start.record()
    for i in range(K):
        align()
        ev_s[i].record(main)
        one_step(timing[i] if timing is not None else None)
        ev_e[i].record(main)
    end.record()
    sync()
    barrier()
    clocks = clk.stop()
    my_ms = start.elapsed_time(end) / K
    step_ms = [a.elapsed_time(b) for a, b in zip(ev_s, ev_e)]
    if timing is not None:
        el = lambda evs, a, b: evs[a].elapsed_time(evs[b])  # noqa: E731
        fwd_ms = sum(el(evs, 0, 1) + el(evs, 2, 3) for per in timing for evs in per) / K
        bwd_ms = sum(el(evs, 4, 5) + el(evs, 6, 7) for per in timing for evs in per) / K
    else:
        kt = {"fwd": 0.0, "bwd": 0.0}
        for rs, _ in steps:
            for kind, a, b in rs.events:
                kt[kind[:3]] += a.elapsed_time(b)
            rs.events = None
        fwd_ms, bwd_ms = kt["fwd"] / K, kt["bwd"] / K

    # ---- e2e: host pinned inputs -> device, step, gradients back to host. Pipelined like a
    # prefetching DataLoader: two device input sets; the H2D of step k+1 and the D2H of step k's
    # gradients (staged by a device copy) run on two copy streams (one per direction of the host link)
    # while step k computes. Every timed step still moves all of its inputs in and all of its
    # gradients out.
    e2e = None
    if not args.no_e2e:
        host = [{k: v.cpu().pin_memory() for k, v in src.items()} for _, src in steps]
        outs = [{k: torch.empty(getattr(rs, k)[:rs.rows].shape, dtype=torch.bfloat16).pin_memory()
                 for k in ("dq", "dk", "dv")} for rs, _ in steps]
        h2d = sum(t.numel() * t.element_size() for hs in host for t in hs.values())
        d2h = sum(t.numel() * t.element_size() for o in outs for t in o.values())
        dev_in = [[{k: torch.empty_like(v) for k, v in src.items()} for _, src in steps] for _ in range(2)]
        # staging for the gradients, double-buffered by step parity (the micro-batches share their
        # working buffers, so each micro-batch's gradients are staged right after its backward)
        stage = [[{k: torch.empty_like(o[k], device="cuda") for k in o} for o in outs] for _ in range(2)]
        copy, copy_out = torch.cuda.Stream(), torch.cuda.Stream()   # one per direction (full duplex)
        # per input set and micro-batch: one event once its Q, K, V are in (the forward may start),
        # one once its dO is in (the backward may start)
        ev_qkv = [[torch.cuda.Event() for _ in range(n_mb)] for _ in range(2)]
        ev_do = [[torch.cuda.Event() for _ in range(n_mb)] for _ in range(2)]
        ev_used = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out_free = [torch.cuda.Event(), torch.cuda.Event()]
        used_rec = [False, False]
        out_rec = [False, False]

        def h2d_set(b):
            with torch.cuda.stream(copy):
                if used_rec[b]:
                    copy.wait_event(ev_used[b])      # the step that last read this set is done
                for m, (hs, di) in enumerate(zip(host, dev_in[b])):
                    for k in ("q", "k", "v"):
                        di[k].copy_(hs[k], non_blocking=True)
                    ev_qkv[b][m].record(copy)
                    di["do"].copy_(hs["do"], non_blocking=True)
                    ev_do[b][m].record(copy)

        def e2e_run(n):
            h2d_set(0)
            for k in range(n):
                b = k % 2
                if k + 1 < n:
                    h2d_set(1 - b)
                if out_rec[b]:
                    main.wait_event(ev_out_free[b])  # the D2H of step k-2 has read this staging set
                for m, ((rs, _), di, st) in enumerate(zip(steps, dev_in[b], stage[b])):
                    main.wait_event(ev_qkv[b][m])
                    fwd_bwd(rs, di, ev_do[b][m])
                    for kk in st:
                        st[kk].copy_(getattr(rs, kk)[:rs.rows], non_blocking=True)
                ev_used[b].record(main)
                used_rec[b] = True
                ev_out[b].record(main)
                with torch.cuda.stream(copy_out):
                    copy_out.wait_event(ev_out[b])
                    for st, o in zip(stage[b], outs):
                        for kk in o:
                            o[kk].copy_(st[kk], non_blocking=True)
                    ev_out_free[b].record(copy_out)
                out_rec[b] = True
            main.wait_event(ev_out_free[0])
            main.wait_event(ev_out_free[1])

        e2e_run(2)
        sync()
        barrier()
        s2, e2_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        e2e_run(K)
        e2_.record()
        sync()
        barrier()
        e2e_ms = s2.elapsed_time(e2_) / K
        e2e = (e2e_ms, h2d, d2h)

    # ---- reduce over ranks: max (headline), per-rank lists (imbalance per step)
    vals = torch.tensor([my_ms, fwd_ms, bwd_ms, e2e[0] if e2e else 0.0] + step_ms, device="cuda",
                        dtype=torch.float64)
    if world > 1:
        if backend != "nccl":
            vals = vals.cpu()                 # gloo moves host tensors
        allv = [torch.zeros_like(vals) for _ in range(world)]
        dist.all_gather(allv, vals)
        allv = torch.stack(allv).cpu().numpy()
    else:
        allv = vals.cpu().numpy()[None]
    loop_ms = float(allv[:, 0].max())
    total_flops = useful_flops(lens, shp)
    value = total_flops / (loop_ms * 1e-3) / 1e12

    if rank == 0:
        per_step = allv[:, 4:]                                  # [ranks, K]
        step_max, step_mean = per_step.max(axis=0), per_step.mean(axis=0)
        imb = step_max / np.maximum(step_mean, 1e-12)
        step_tflops = total_flops / (step_max * 1e-3) / 1e12
        peaks, which = measured_peaks()
        (peak, peak_key), burst, sus = pick_peak(peaks, clocks, loop_ms * K / 1e3)
        # dominant kernel: the forward or backward attention calls of rank 0 (algorithmic flops of
        # this rank: 4 / 10 * d * Hq per causal pair it computes), timed inside the headline loop
        my_pairs = sum(rank_pairs(ml, ma, cp, cp_rank) for ml, ma in mbs)
        fwd_fl, bwd_fl = 4 * shp.d * shp.hq * my_pairs, 10 * shp.d * shp.hq * my_pairs
        my_fwd, my_bwd = float(allv[0, 1]), float(allv[0, 2])
        dom = ("bwd", bwd_fl, my_bwd) if my_bwd >= my_fwd else ("fwd", fwd_fl, my_fwd)
        achieved = dom[1] / (dom[2] * 1e-3) / 1e12
        traffic = ncu_traffic(name, world, dom[0])
        launches_per_step = sum(rs.launches_per_step(args.exchange) for rs, _ in steps)
        gpu_launches = K * launches_per_step
        cpu = None
        if not args.no_cpu_baseline and world == 1:   # the oracle baseline is an N=1 figure
            v, n, toks, t, _ = cpu_oracle_sample(lens, shp, args.cpu_seconds, args.seed)
            cpu = {"value": v, "unit": "TFLOP/s", "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
                   "sample": f"{n} shortest sequences ({toks} tokens) of the batch, fp64 numpy fwd+bwd, {t:.1f} s"}
        # the Python scheduler oracle (exact Fractions, Alg. 1-3 + LPT) on the same global batch,
        # beside the C++ skr_plan (SURVEY §8(d) "Oracle timing beside the GPU path")
        from oracle.cost_model import Model
        from oracle.schedule import plan as oracle_plan
        t0 = time.perf_counter()
        ref = oracle_plan([int(x) for x in lens], int(bucket), cp, dp, Model(h, hkv))
        oracle_plan_us = (time.perf_counter() - t0) * 1e6
        assert list(ref.assign) == list(plan["assign"]), "skr_plan differs from the scheduler oracle"
        # plan floor (Eq. 8 style): per DP rank, sum over its micro-batches of the slowest CP rank's
        # causal pairs; the slowest DP rank over the mean pairs per GPU
        t_dp, tot = [], 0
        for d_mbs in all_mbs:
            pp = [[rank_pairs(ml, ma, cp, r) for r in range(cp)] for ml, ma in d_mbs]
            t_dp.append(sum(max(p) for p in pp))
            tot += sum(sum(p) for p in pp)
        floor = max(t_dp) / max(1e-9, tot / world)
        predicted = eval_prediction(sk, all_mbs, cp, bucket, shp)
        attn_ms = my_fwd + my_bwd
        out = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": loop_ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": name, "desc": cfg.note if (world == 1 or name != "C2") else f"{cfg.note}; weak-scaled x{world}",
                       "shape": f"Hq={shp.hq} Hkv={shp.hkv} d={shp.d}", "global_batch": int(len(lens)),
                       "tokens": int(lens.sum()), "max_seq_len": int(lens.max()), "cp": cp, "dp": dp,
                       "bucket_tokens": int(bucket), "micro_batches": n_mb,
                       "distributed_seqs": int((plan["assign"] == -1).sum()),
                       "rollbacks": int(plan["n_rollbacks"]),
                       "l2": "inputs larger than L2 (no flush)",
                       "parallelism": f"dp{dp}xcp{cp}" if dp > 1 else f"cp{cp}",
                       "exchange": args.exchange if cp > 1 else None,
                       "bwd_band_rows": int(sk.skr_attn_bwd_band_rows(shape) if args.bwd_band is None else args.bwd_band)},
            "roofline": {"bound": "tensor", "kernel": f"attn_{dom[0]} calls (rank 0, inside the timed loop; "
                                                      f"bwd includes its D-preprocess and dQ convert)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "frac_of_burst": achieved / burst, "frac_of_sustained": achieved / sus,
                         "traffic": traffic[0] if traffic else None,
                         "traffic_source": traffic[1] if traffic else None,
                         "peak_source": f"{which} {peak_key} (MEASURED_PEAKS.json); sustained applies when the "
                                        f"timed region is >= 2 s at power-capped clocks"},
            "cpu_baseline": cpu,
            "e2e": None if e2e is None else {"value": total_flops / (float(allv[:, 3].max()) * 1e-3) / 1e12,
                                             "unit": "TFLOP/s", "h2d_bytes_per_step": e2e[1],
                                             "d2h_bytes_per_step": e2e[2],
                                             "pipeline": "H2D of step k+1 and D2H of step k overlap step k"},
            "gpu_launches": gpu_launches,
            "clocks": clocks,
            "max_mean_rank_time": float(np.median(imb)),
            "max_mean_rank_time_p10_p90": [pctl(imb, 10), pctl(imb, 90)],
            "step_tflops_median": float(np.median(step_tflops)),
            "step_tflops_p10_p90": [pctl(step_tflops, 10), pctl(step_tflops, 90)],
            "plan_floor": floor,
            "eval_predicted_ms": predicted,
            "plan_us": plan_us, "plan_us_oracle_python": oracle_plan_us,
            "fwd_ms": float(allv[:, 1].max()), "bwd_ms": float(allv[:, 2].max()),
            "rest_of_step_ms": loop_ms - attn_ms,
            "rest_of_step": "pack Q/K/V/dO, K/V exchange waits, dK/dV partial zeroing, launch gaps and the "
                            "per-step rank alignment (rank 0)",
        }
        print(json.dumps(out), flush=True)
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
