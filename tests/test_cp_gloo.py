"""Multi-process CPU test (gloo, world size 2 and 3) of the CP exchange logic (rows a4/a6/a9).

Every rank computes the plan with the C-ABI host planner (identical on all ranks, no
communication), builds its pack tables, and moves row identities through REAL collectives:
  forward : packed distributed prefix (P rows) -> all_gather -> chunk-table reorder -> must equal
            the natural per-sequence order of every distributed sequence (R20-R23);
  backward: per-rank partial "gradients" in natural order -> chunk-table permute to rank-major ->
            reduce_scatter(sum) -> each rank's result must equal the sum over ranks for exactly the
            rows of its own distributed prefix.
The table application is emulated with numpy here (the device kernels are checked on the GPU).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

LENS = [3, 700, 17, 1500, 64, 5, 900, 2, 300, 1200, 33]
SHAPE = (8, 2, 64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world_size, port, C, q, dp=1):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world_size)
        from paper_2505_19609_b200 import skrull as sk
        from paper_2505_19609_b200.runtime import dp_micro_batches, grid_coords, rank_natural_rows
        hq, hkv, d = SHAPE
        lens = np.asarray(LENS, np.int64)
        # DP x CP grid (row f4): this rank's CP group = `world` consecutive ranks
        dp_rank, rank, world = grid_coords(rank, world_size, dp)
        groups = [dist.new_group(list(range(g * world, (g + 1) * world))) for g in range(dp)]
        grp = groups[dp_rank]
        p = sk.skr_plan(lens, C, world, dp, hq * d, hkv * d)
        # identical plans on every rank
        mine = torch.tensor(np.concatenate([p["assign"], p["mb_of_seq"], p["dp_of_seq"]]), dtype=torch.int64)
        allp = [torch.zeros_like(mine) for _ in range(world_size)]
        dist.all_gather(allp, mine)
        assert all(torch.equal(x, mine) for x in allp)
        n_dist_total = 0
        for idx, ml, ma in dp_micro_batches(p, lens, dp_rank):
            pr = sk.skr_pack_rank(ml, ma, world, rank)
            if pr["natural_rows"] == 0:
                continue
            n_dist_total += int((ma == -1).sum())
            table = sk.skr_pack_chunks(ml, ma, world)
            P = pr["pad_rows_P"]
            # identity of each row = seq * 2^20 + position
            src = np.array([k * (1 << 20) + pos for k, lo, hi in rank_natural_rows(ml, ma, world, rank)
                            for pos in range(lo, hi)], np.int64)
            packed = src[pr["src_row"]]
            send = np.full(P, -1, np.int64)
            n = min(P, len(packed))
            send[:n] = packed[:n]
            gathered = [torch.zeros(P, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(send), group=grp)
            g = torch.cat(gathered).numpy()
            natural = np.full(pr["natural_rows"], -2, np.int64)
            for seq, c, owner, grow, nrow, ln in table:
                natural[nrow:nrow + ln] = g[grow:grow + ln]
            expect = np.concatenate([k * (1 << 20) + np.arange(ml[k]) for k in np.argsort(ml, kind="stable")
                                     if ma[k] == -1])
            assert np.array_equal(natural, expect), "all-gather + reorder does not rebuild natural K/V order"
            # backward: partial = (rank + 1) * identity; reduce-scatter the rank-major permutation
            partial = (rank + 1) * natural.astype(np.float64)
            rm = np.zeros(world * P)
            for seq, c, owner, grow, nrow, ln in table:
                rm[grow:grow + ln] = partial[nrow:nrow + ln]
            out = torch.zeros(P, dtype=torch.float64)
            dist.reduce_scatter(out, list(torch.from_numpy(rm).chunk(world)), group=grp)
            tot = sum(r + 1 for r in range(world))
            dr = pr["dist_rows"]
            assert np.array_equal(out.numpy()[:dr], tot * packed[:dr].astype(np.float64)), \
                "reduce-scatter does not land on the rank's own distributed prefix"
        q.put((rank, "ok", n_dist_total))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world,C,dp", [(2, 1800, 1), (3, 1300, 1), (4, 1100, 2)])
def test_cp_exchange_tables_over_gloo(world, C, dp):
    # (4, 1100, 2): a DP=2 x CP=2 grid, the exchange inside each CP group's sub-communicator
    pytest.importorskip("paper_2505_19609_b200.skrull")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, C, q, dp)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, status, info in res:
        assert status == "ok", f"rank {rank}: {info}"
    assert all(info > 0 for _, _, info in res), "the test plan must shard at least one sequence"
