"""GPU: the CP runtime (pack -> K/V exchange -> fwd local/dist -> bwd dist/local -> dK/dV exchange)
for N ranks driven on ONE GPU with a loopback exchange (SURVEY §4 debug aid), checked against the
unsharded fp64 oracle: sharded == unsharded for every sequence, every output.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.attention import attn_bwd, attn_fwd  # noqa: E402
from oracle.schedule import plan as oracle_plan  # noqa: E402
from oracle.cost_model import Model  # noqa: E402
from tests.attn_harness import make_inputs, tol_ok  # noqa: E402


def _baseline_plan(sk, lens, C, N, planner):
    """Row f1: the paper's baselines as plans the same runtime executes (one DP rank). 'rr' /
    'rr_norb': Alg. 4 round-robin with / without roll-back (R27) on one micro-batch;
    'full_shard': FIFO micro-batches under C*N (Eq. 10), every sequence distributed (the
    DeepSpeed-like CP of P:101). Bit-exact against the oracle's implementations."""
    from oracle.schedule import ScheduleError, full_shard, round_robin
    K = len(lens)
    if planner in ("rr", "rr_norb"):
        rb = planner == "rr"
        try:
            ref = round_robin(list(lens), C, N, rb)
        except ScheduleError:
            with pytest.raises(sk.SkrullError):
                sk.skr_round_robin(lens, C, N, rb)
            return None
        A, _ = sk.skr_round_robin(lens, C, N, rb)
        assert list(A) == ref                                     # bit-exact baseline plan
        return dict(dp_of_seq=np.zeros(K, np.int32), mb_of_seq=np.zeros(K, np.int32), assign=np.asarray(A),
                    n_mb_per_dp=np.asarray([1], np.int32), n_rollbacks=0)
    mbs = full_shard(list(lens), C, N)
    M, n = sk.skr_full_shard(lens, C, N)
    assert n == len(mbs) and all(M[k] == j for j, mb in enumerate(mbs) for k in mb)
    return dict(dp_of_seq=np.zeros(K, np.int32), mb_of_seq=np.asarray(M), assign=np.full(K, -1, np.int32),
                n_mb_per_dp=np.asarray([n], np.int32), n_rollbacks=0)


def _run(lens, hq, hkv, d, N, C, bf16, seed, dp=1, exchange="nccl", planner="skrull"):
    from paper_2505_19609_b200 import skrull as sk
    from paper_2505_19609_b200.runtime import (RankStep, dp_micro_batches, gather_rank_natural, loopback_peer_fused_step,
                                               loopback_peer_step, loopback_ring_step, loopback_step)
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16 if bf16 else sk.SKR_FP32)
    if planner == "skrull":
        p = sk.skr_plan(lens, C, N, dp, hq * d, hkv * d)
        ref = oracle_plan(list(lens), C, N, dp, Model(hq * d, hkv * d))
        assert list(p["assign"]) == ref.assign                       # bit-exact plan
        assert list(p["dp_of_seq"]) == ref.dp_of_seq and list(p["mb_of_seq"]) == ref.mb_of_seq
    else:
        assert dp == 1
        p = _baseline_plan(sk, lens, C, N, planner)
        if p is None:                                   # the baseline fails (Table 3 "OOM"), as the oracle does
            return None, None
    inputs = make_inputs(lens, hq, hkv, d, seed=seed, bf16=bf16)
    tdt = torch.bfloat16 if bf16 else torch.float32
    src_key = {"o": "q", "dq": "q", "dk": "k", "dv": "k"}
    outs = {k: [np.full((int(S),) + x[src_key[k]].shape[1:], np.nan) for S, x in zip(lens, inputs)]
            for k in ("o", "dq", "dk", "dv")}
    lse = [np.full((hq, int(S)), np.nan) for S in lens]
    n_dist = 0
    for idx, ml, ma in [mb for dr in range(dp) for mb in dp_micro_batches(p, lens, dr)]:
        n_dist += int((ma == -1).sum())
        mb_inputs = [inputs[i] for i in idx]
        ranks = [RankStep(shape, ml, ma, N, r, ring=exchange == "ring") for r in range(N)]
        srcs = {k: [torch.from_numpy(gather_rank_natural(mb_inputs, ml, ma, N, r, k)).to("cuda", tdt)
                    for r in range(N)] for k in ("q", "k", "v", "do")}
        step = {"peer": loopback_peer_step, "fused": loopback_peer_fused_step,
                "ring": loopback_ring_step}.get(exchange, loopback_step)
        step(ranks, srcs["q"], srcs["k"], srcs["v"], srcs["do"])
        torch.cuda.synchronize()
        for r, rs in enumerate(ranks):
            pr = rs.pr
            f = lambda t: t.float().cpu().numpy()  # noqa: E731
            o, dq, dk, dv, L = f(rs.o), f(rs.dq), f(rs.dk), f(rs.dv), f(rs.lse)
            for i in range(pr["n_seg"]):
                a, b = pr["cu_seqlens_q"][i], pr["cu_seqlens_q"][i + 1]
                s = idx[pr["seg_seq"][i]]
                lo = pr["q_pos"][i]
                for key, arr in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
                    outs[key][s][lo:lo + b - a] = arr[a:b]
                lse[s][:, lo:lo + b - a] = L[:, a:b]
    for s, x in enumerate(inputs):
        O, Lr = attn_fwd(x["q"], x["k"], x["v"])
        dQ, dK, dV = attn_bwd(x["q"], x["k"], x["v"], x["do"])
        for key, ref in (("o", O), ("dq", dQ), ("dk", dK), ("dv", dV)):
            got = outs[key][s]
            assert not np.isnan(got).any(), f"{key} seq {s}: rows not covered"
            ok, err, bound = tol_ok(got, ref, not bf16, label=f"{key} cp")
            assert ok, f"{key} seq {s} (len {lens[s]}, N={N}): err {err} > {bound}"
        assert np.abs(lse[s] - Lr).max() <= (2e-2 if bf16 else 1e-5 * max(1, np.abs(Lr).max()))
    return n_dist, p


def test_toy_c1_fp32_cp2():
    # BASELINE configs[0]: toy 8 sequences, 2 heads, d=64, fp32, CP=2 plan (C=600): 3 distributed
    n_dist, p = _run([17, 33, 64, 90, 128, 200, 256, 300], 2, 2, 64, 2, 600, False, 0)
    assert n_dist == 3 and p["n_rollbacks"] == 2


def test_toy_c1_gqa_fp32_cp2():
    _run([17, 33, 64, 90, 128, 200, 256, 300], 2, 1, 64, 2, 600, False, 1)


@pytest.mark.parametrize("N", [2, 4])
def test_bf16_cp_mixed(N):
    # long + short mix with C below the longest sequence (R33): the long ones are sharded
    lens = [1500, 37, 300, 129, 1, 600, 64, 2000, 250]
    C = 1600 if N == 2 else 900
    n_dist, _ = _run(lens, 8, 2, 128, N, C, True, 2)
    assert n_dist >= 1


def test_bf16_cp_d64_rollback_cascade():
    # tiny sequences rolled back into distributed status: chunks of 0-2 tokens (S < 2N)
    lens = [3, 5, 2, 700, 800, 1, 7]
    n_dist, p = _run(lens, 14, 2, 64, 4, 400, True, 3)
    assert n_dist >= 2


def test_n1_all_local():
    lens = [1, 17, 300, 129, 1024]
    n_dist, p = _run(lens, 14, 2, 64, 1, 4096, True, 4)
    assert n_dist == 0


def test_dp2_x_cp2_grid():
    # row f4: DP x CP grid (GDS/LPT bins over 2 DP ranks, DACP inside each CP group of 2); every DP
    # rank's micro-batches run through its own CP group (loopback), all sequences covered once
    lens = [1500, 37, 300, 129, 1, 600, 64, 2000, 250, 900, 17, 1100]
    n_dist, p = _run(lens, 8, 2, 128, 2, 1200, True, 5, dp=2)
    assert set(p["dp_of_seq"]) == {0, 1} and n_dist >= 1


@pytest.mark.parametrize("exchange", ["peer", "fused", "ring"])
@pytest.mark.parametrize("case", ["c1_fp32", "bf16_n2", "bf16_n4", "rollback_d64"])
def test_peer_exchange_loopback(case, exchange):
    # row f3: the a6 / a9 exchange as peer-gather / peer-reduce kernels (one pass each, "peer") or
    # with the a9 reduction fused into the distributed backward kernel's epilogue ("fused", step
    # two) instead of all-gather + reorder and permute + reduce-scatter + cast; row f4: ring CP
    # ("ring": K/V hops, partial attentions merged, travelling dK/dV accumulators); same oracle bar
    lens = [1500, 37, 300, 129, 1, 600, 64, 2000, 250]
    if case == "c1_fp32":
        n_dist, _ = _run([17, 33, 64, 90, 128, 200, 256, 300], 2, 2, 64, 2, 600, False, 0, exchange=exchange)
    elif case == "bf16_n2":
        n_dist, _ = _run(lens, 8, 2, 128, 2, 1600, True, 2, exchange=exchange)
    elif case == "bf16_n4":
        n_dist, _ = _run(lens, 8, 2, 128, 4, 900, True, 2, exchange=exchange)
    else:
        n_dist, _ = _run([3, 5, 2, 700, 800, 1, 7], 14, 2, 64, 4, 400, True, 3, exchange=exchange)
    assert n_dist >= 1


def test_buffer_pool_micro_batches_share_buffers():
    # GDS splits this batch into several micro-batches; their RankSteps take views of ONE BufferPool
    # (bench.py's memory layout) and run one after another through the composite C-ABI step
    # (skr_cp_attn_fwd / _bwd, N = 1); each micro-batch is read back right after its backward.
    from paper_2505_19609_b200 import skrull as sk
    from paper_2505_19609_b200.runtime import BufferPool, RankStep, gather_rank_natural
    lens = [900, 37, 700, 129, 1, 600, 64, 1000, 250, 333]
    hq, hkv, d = 8, 2, 64
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
    p = sk.skr_plan(lens, 1200, 1, 1, hq * d, hkv * d)
    n_mb = int(p["n_mb_per_dp"][0])
    assert n_mb >= 3
    inputs = make_inputs(lens, hq, hkv, d, seed=9, bf16=True)
    pool = BufferPool()
    mbs = []
    for j in range(n_mb):
        idx = np.nonzero(p["mb_of_seq"] == j)[0]
        ml, ma = np.asarray(lens)[idx], p["assign"][idx]
        mbs.append((idx, ml, ma, RankStep(shape, ml, ma, 1, 0, alloc=pool.reserve)))
    pool.materialize()
    for *_, rs in mbs:
        rs.rebind(pool.get)
    assert len({rs.q.data_ptr() for *_, rs in mbs}) == 1          # one shared working set
    for idx, ml, ma, rs in mbs:
        mb_inputs = [inputs[i] for i in idx]
        src = {k: torch.from_numpy(gather_rank_natural(mb_inputs, ml, ma, 1, 0, k)).to("cuda", torch.bfloat16)
               for k in ("q", "k", "v", "do")}
        rs.forward(src["q"], src["k"], src["v"])
        rs.backward(src["do"])
        torch.cuda.synchronize()
        pr = rs.pr
        for i in range(pr["n_seg"]):
            a, b = pr["cu_seqlens_q"][i], pr["cu_seqlens_q"][i + 1]
            x = inputs[idx[pr["seg_seq"][i]]]
            O, _ = attn_fwd(x["q"], x["k"], x["v"])
            dQ, dK, dV = attn_bwd(x["q"], x["k"], x["v"], x["do"])
            for key, ref in (("o", O), ("dq", dQ), ("dk", dK), ("dv", dV)):
                ok, err, bound = tol_ok(getattr(rs, key)[a:b].float().cpu().numpy(), ref, False, label=f"{key} pool")
                assert ok, f"{key} seq {idx[pr['seg_seq'][i]]}: err {err} > {bound}"


@pytest.mark.parametrize("case", range(24))
def test_random_plans_fuzz(case):
    # randomised end-to-end parity: random GQA shape, head dim, CP degree, Long-SFT-like lengths and a
    # BucketSize between the feasibility bound and no sharding; every output against the fp64 oracle.
    # (Cases 6 and 11 found that padding rows past a rank's own rows -- read by the 128-row tiles and
    # multiplied by exact zeros -- must be finite: the runtime now zero-fills its buffers.)
    import random
    rng = random.Random(1000 + case)
    hkv = rng.choice([1, 2, 4])
    hq = hkv * rng.choice([1, 2, 3, 7])
    d = rng.choice([64, 128])
    N = rng.choice([1, 2, 3, 4])
    K = rng.randint(2, 9)
    lens = [int(min(3000, max(1, rng.lognormvariate(5.0, 1.4)))) for _ in range(K)]
    lo = max(max(lens) // N + 1, 64)
    C = rng.randint(lo, max(lo, sum(lens) // N + 256))
    # every 6th case in fp32 test mode; a quarter of the cases through each exchange: all-gather /
    # reduce-scatter, the row-f3 peer-memory exchange (step one), its fused step two, the row-f4 ring
    _run(lens, hq, hkv, d, N, C, case % 6 != 5, 50 + case,
         exchange={0: "nccl", 1: "peer", 2: "fused", 3: "ring"}[case % 4])


@pytest.mark.parametrize("planner", ["rr", "rr_norb", "full_shard"])
@pytest.mark.parametrize("case", range(6))
def test_baseline_plans_fuzz(planner, case):
    # row f1: the baselines' plans (round-robin Alg. 4 with / without roll-back, full-shard CP)
    # through the same CP runtime and kernels, every output against the fp64 oracle
    import random
    rng = random.Random(2000 + case)
    hkv = rng.choice([1, 2])
    hq = hkv * rng.choice([1, 3, 7])
    d = rng.choice([64, 128])
    N = rng.choice([2, 3, 4])
    K = rng.randint(3, 9)
    lens = [int(min(2500, max(1, rng.lognormvariate(5.0, 1.4)))) for _ in range(K)]
    lo = max(max(lens) // N + 1, 64)
    C = rng.randint(lo, max(lo, sum(lens) // N + 256))
    if planner != "full_shard":
        C = max(C, -(-sum(lens) // N) + 8)   # round-robin plans one micro-batch: Eq. 10 must hold
    n_dist, p = _run(lens, hq, hkv, d, N, C, case % 3 != 2, 80 + case, planner=planner)
    if p is not None and planner == "full_shard":
        assert n_dist == K
