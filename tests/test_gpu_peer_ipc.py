"""GPU, two processes: row f3's peer-memory CP exchange across PROCESSES with real CUDA IPC mappings
and the epoch flags, on one B200 (both ranks on cuda:0 -- IPC between processes of the same device
is the same mechanism that maps a peer GPU's memory over NVLink). gloo carries the control plane
(IPC blobs); the data plane is the library's peer-gather / peer-reduce / signal / wait kernels.
Each rank runs forward_peer + backward_peer (step one: peer-reduce pass) or backward_peer_fused
(step two: the backward kernel red-adds dK/dV into the owners' accumulators in the other process)
of its CP rank; the parent checks every output against the fp64 oracle (sharded == unsharded)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.multiprocessing as mp  # noqa: E402

LENS = [3000, 37, 300, 129, 1, 600, 64, 250]
HQ, HKV, D, C, SEED = 8, 2, 128, 2400, 2      # one micro-batch: 3000, 1 and 64 sharded, the rest local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, mode):
    import torch.distributed as dist
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2505_19609_b200 import skrull as sk
        from paper_2505_19609_b200.runtime import RankStep, gather_rank_natural
        from tests.attn_harness import make_inputs
        shape = sk.attn_shape(HQ, HKV, D, sk.SKR_BF16)
        lens = np.asarray(LENS, np.int64)
        p = sk.skr_plan(lens, C, world, 1, HQ * D, HKV * D)
        assert int(p["n_mb_per_dp"][0]) == 1
        assign = p["assign"]
        inputs = make_inputs(lens, HQ, HKV, D, seed=SEED, bf16=True)
        peer = sk.PeerComm(world, rank)
        rs = RankStep(shape, lens, assign, world, rank)
        rs.connect_peer(peer)
        src = {k: torch.from_numpy(gather_rank_natural(inputs, lens, assign, world, rank, k)).to("cuda", torch.bfloat16)
               for k in ("q", "k", "v", "do")}
        side = torch.cuda.Stream()
        for _ in range(2):                      # twice: the epochs must also order buffer reuse
            rs.forward_peer(src["q"], src["k"], src["v"], side)
            (rs.backward_peer_fused if mode == "fused" else rs.backward_peer)(src["do"], side)
        torch.cuda.synchronize()
        peer.check()
        f = lambda t: t[:rs.rows].float().cpu().numpy()  # noqa: E731
        q.put((rank, "ok", dict(pr=rs.pr, o=f(rs.o), dq=f(rs.dq), dk=f(rs.dk), dv=f(rs.dv),
                                n_dist=int((assign == -1).sum()))))
        dist.barrier()                          # peers stay mapped until every rank is done
        peer.close()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["step1", "fused"])
def test_peer_exchange_two_processes(mode):
    from oracle.attention import attn_bwd, attn_fwd
    from tests.attn_harness import make_inputs, tol_ok
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
    for rank, status, info in res:
        assert status == "ok", f"rank {rank}: {info}"
    assert res[0][2]["n_dist"] >= 1
    inputs = make_inputs(LENS, HQ, HKV, D, seed=SEED, bf16=True)
    outs = {k: [np.full((S,) + inputs[i]["q" if k in ("o", "dq") else "k"].shape[1:], np.nan)
                for i, S in enumerate(LENS)] for k in ("o", "dq", "dk", "dv")}
    for rank, _, r in res:
        pr = r["pr"]
        for i in range(pr["n_seg"]):
            a, b = pr["cu_seqlens_q"][i], pr["cu_seqlens_q"][i + 1]
            s, lo = pr["seg_seq"][i], pr["q_pos"][i]
            for key in ("o", "dq", "dk", "dv"):
                outs[key][s][lo:lo + b - a] = r[key][a:b]
    for s, x in enumerate(inputs):
        O, _ = attn_fwd(x["q"], x["k"], x["v"])
        dQ, dK, dV = attn_bwd(x["q"], x["k"], x["v"], x["do"])
        for key, ref in (("o", O), ("dq", dQ), ("dk", dK), ("dv", dV)):
            got = outs[key][s]
            assert not np.isnan(got).any(), f"{key} seq {s}: rows not covered"
            ok, err, bound = tol_ok(got, ref, False, label=f"{key} peer-ipc-{mode}")
            assert ok, f"{key} seq {s} (len {LENS[s]}): err {err} > {bound}"
