"""GPU: the NCCL data plane of rows a6 / a9 through the composite C-ABI step.

skr_cp_attn_fwd / skr_cp_attn_bwd with a LIVE skr_comm run the production exchange: the grouped
ncclAllGather of the packed K / V distributed prefix on the side stream, the reorder to natural
order, the fp32 permute, the grouped ncclReduceScatter (sum) and the cast into the packed dK / dV
prefix, with the cross-stream events of Eq. 2's overlap (mirrored for the backward,
reading R24). On one GPU the CP group is a 1-rank NCCL communicator and the distributed sequences
are HAND-assigned (assign = -1 at cp = 1 splits a sequence into zigzag chunks 0 and 1, both on rank
0: the all-gather and reduce-scatter then move real data through NCCL, one rank wide). Every
output is checked against the unsharded fp64 oracle (tolerance R34', tests/attn_harness.tol_ok).
A 2-rank variant (two processes, real NCCL over two GPUs) runs when two GPUs are visible.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.attention import attn_bwd, attn_fwd  # noqa: E402
from tests.attn_harness import make_inputs, tol_ok  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_nccl_step(lens, assign, hq, hkv, d, bf16, seed, cp=1, rank=0, comm=None, reps=1, ring=False):
    """One micro-batch on CP rank `rank` through skr_cp_attn_fwd / _bwd with `comm` (a 1-rank
    communicator when None), or with ring=True through the row-f4 ring CP (forward_ring /
    backward_ring: NCCL point-to-point hops). Returns the per-sequence outputs this rank owns:
    {seq: {key: (q_lo, array)}} plus the RankStep."""
    from paper_2505_19609_b200 import skrull as sk
    from paper_2505_19609_b200.runtime import RankStep, gather_rank_natural
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16 if bf16 else sk.SKR_FP32)
    inputs = make_inputs(lens, hq, hkv, d, seed=seed, bf16=bf16)
    tdt = torch.bfloat16 if bf16 else torch.float32
    own = comm is None
    if own:
        comm = sk.Comm(1, 0)
    assert comm.size() == (cp, rank)
    rs = RankStep(shape, np.asarray(lens), np.asarray(assign, np.int32), cp, rank, ring=ring)
    src = {k: torch.from_numpy(gather_rank_natural(inputs, lens, assign, cp, rank, k)).to("cuda", tdt)
           for k in ("q", "k", "v", "do")}
    side = torch.cuda.Stream(priority=-1)
    for _ in range(reps):      # repeated steps reuse every buffer (the bench's steady state)
        if ring:
            rs.forward_ring(src["q"], src["k"], src["v"], comm, side)
            rs.backward_ring(src["do"], comm, side)
        else:
            rs.forward(src["q"], src["k"], src["v"], comm, side)
            rs.backward(src["do"], comm, side)
    comm.wait(torch.cuda.current_stream(), timeout_s=120.0)     # polls ncclCommGetAsyncError
    comm.check()
    torch.cuda.synchronize()
    out = {}
    pr = rs.pr
    f = lambda t: t.float().cpu().numpy()  # noqa: E731
    o, dq, dk, dv, L = f(rs.o), f(rs.dq), f(rs.dk), f(rs.dv), f(rs.lse)
    for i in range(pr["n_seg"]):
        a, b = int(pr["cu_seqlens_q"][i]), int(pr["cu_seqlens_q"][i + 1])
        s = int(pr["seg_seq"][i])
        lo = int(pr["q_pos"][i])
        e = out.setdefault(s, [])
        e.append((lo, {"o": o[a:b], "dq": dq[a:b], "dk": dk[a:b], "dv": dv[a:b], "lse": L[:, a:b]}))
    if own:
        comm.close()
    return inputs, out, rs


def check_against_oracle(inputs, per_rank_outs, lens, bf16):
    for s, x in enumerate(inputs):
        S = int(lens[s])
        got = {k: np.full((S,) + x["q" if k in ("o", "dq") else "k"].shape[1:], np.nan) for k in ("o", "dq", "dk", "dv")}
        lse = np.full((x["q"].shape[1], S), np.nan)
        for out in per_rank_outs:
            for lo, parts in out.get(s, []):
                n = parts["o"].shape[0]
                for k in got:
                    got[k][lo:lo + n] = parts[k]
                lse[:, lo:lo + n] = parts["lse"]
        O, Lr = attn_fwd(x["q"], x["k"], x["v"])
        dQ, dK, dV = attn_bwd(x["q"], x["k"], x["v"], x["do"])
        for key, ref in (("o", O), ("dq", dQ), ("dk", dK), ("dv", dV)):
            assert not np.isnan(got[key]).any(), f"{key} seq {s}: rows not covered"
            ok, err, bound = tol_ok(got[key], ref, not bf16, label=f"{key} nccl")
            assert ok, f"{key} seq {s} (len {S}): err {err} > {bound}"
        assert np.abs(lse - Lr).max() <= (2e-2 if bf16 else 1e-5 * max(1, np.abs(Lr).max()))


CASES = {
    # (lens, assign, hq, hkv, d, bf16): mixes of hand-distributed (-1) and local (0) sequences
    "bf16_d128": ([1500, 37, 300, 129, 1, 600, 64, 2000, 250], [-1, 0, -1, 0, -1, 0, 0, -1, 0], 8, 2, 128, True),
    "bf16_d64_gqa7": ([1100, 17, 777, 3, 256], [-1, 0, -1, -1, 0], 14, 2, 64, True),
    "fp32_toy_c1": ([17, 33, 64, 90, 128, 200, 256, 300], [-1, 0, -1, 0, 0, 0, 0, -1], 2, 2, 64, False),
    "bf16_all_distributed": ([513, 1024, 2, 129], [-1, -1, -1, -1], 4, 4, 64, True),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_nccl_exchange_one_rank(case):
    lens, assign, hq, hkv, d, bf16 = CASES[case]
    inputs, out, rs = run_nccl_step(lens, assign, hq, hkv, d, bf16, seed=31, reps=2)
    assert rs.has_dist and rs.n_chunks == 2 * sum(1 for a in assign if a == -1)
    check_against_oracle(inputs, [out], lens, bf16)


@pytest.mark.parametrize("case", sorted(CASES))
def test_nccl_ring_one_rank(case):
    # row f4's ring CP on a 1-rank communicator: the hop-0 partial attentions (diagonal and full
    # chunk pairs, the merge) and the travelling dK/dV accumulators' hop through ncclSend / ncclRecv
    # to itself; two steps (buffer reuse)
    lens, assign, hq, hkv, d, bf16 = CASES[case]
    inputs, out, rs = run_nccl_step(lens, assign, hq, hkv, d, bf16, seed=33, reps=2, ring=True)
    assert rs.ring
    check_against_oracle(inputs, [out], lens, bf16)


def test_comm_rank_count_mismatch_is_rejected():
    # a step planned for CP = 2 must not run on a 1-rank communicator (ADVICE: cp_step.cu nranks check)
    from paper_2505_19609_b200 import skrull as sk
    from paper_2505_19609_b200.runtime import RankStep
    shape = sk.attn_shape(4, 2, 64, sk.SKR_BF16)
    rs = RankStep(shape, np.asarray([300, 40]), np.asarray([-1, 0], np.int32), 2, 0)
    comm = sk.Comm(1, 0)
    z = torch.zeros(max(rs.rows, 1), 4, 64, device="cuda", dtype=torch.bfloat16)
    zk = torch.zeros(max(rs.rows, 1), 2, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(sk.SkrullError, match="communicator has 1 ranks"):
        rs.forward(z, zk, zk, comm, torch.cuda.Stream())
    comm.close()


def test_comm_wait_returns_on_idle_stream():
    from paper_2505_19609_b200 import skrull as sk
    comm = sk.Comm(1, 0)
    comm.wait(torch.cuda.current_stream(), timeout_s=5.0)
    comm.check()
    comm.close()


_TWO_RANK = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
from tests.test_gpu_nccl import CASES, run_nccl_step
from paper_2505_19609_b200 import skrull as sk
rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
comm = sk.Comm(2, rank, group=dist.group.WORLD, src=0)
lens, assign, hq, hkv, d, bf16 = CASES[os.environ["CASE"]]
inputs, out, rs = run_nccl_step(lens, assign, hq, hkv, d, bf16, seed=31, cp=2, rank=rank, comm=comm, reps=2,
                                ring=os.environ.get("RING") == "1")
np.save(os.path.join(os.environ["OUT"], f"r{rank}.npy"), np.array([out], dtype=object), allow_pickle=True)
comm.close()
dist.destroy_process_group()
'''


@pytest.mark.parametrize("ring", [False, True])
@pytest.mark.parametrize("case", ["bf16_d128", "fp32_toy_c1"])
def test_nccl_exchange_two_ranks(case, ring, tmp_path):
    # the same hand-assigned step over a real 2-rank NCCL communicator (2 GPUs), both ranks' outputs
    # together against the oracle; skipped on a 1-GPU box
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, ROOT=ROOT, CASE=case, OUT=str(tmp_path), MASTER_ADDR="127.0.0.1", MASTER_PORT="29561",
               WORLD_SIZE="2", RING="1" if ring else "0")
    procs = [subprocess.Popen([sys.executable, "-c", _TWO_RANK], env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              cwd=ROOT) for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    outs = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True)[0] for r in range(2)]
    lens, assign, hq, hkv, d, bf16 = CASES[case]
    check_against_oracle(make_inputs(lens, hq, hkv, d, seed=31, bf16=bf16), outs, lens, bf16)
