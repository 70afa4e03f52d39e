"""Pins for oracle/pack.py (readings R20-R23) and oracle/metrics.py (R32, plan floor)."""
import random

from oracle.metrics import causal_pairs, plan_floor, rank_pairs, useful_flops
from oracle.pack import chunk_bounds, chunk_owner, pack_microbatch
from oracle.schedule import dacp
from oracle.cost_model import Model


def test_toy_pack_hand_trace(golden):
    g = golden("toy_c1_plan.json")
    L, A, N = g["lengths"], g["assign"], g["N"]
    p = pack_microbatch(L, A, N)
    for j, key in enumerate(("rank0", "rank1")):
        r = p.ranks[j]
        assert r.cu_seqlens_q == g[key]["cu_seqlens_q"]
        assert r.q_pos == g[key]["q_pos"]
        assert r.k_len == g[key]["k_len"]
    assert p.pad_rows == g["pad_rows_P"]
    assert p.natural_rows == g["natural_rows"]
    assert {str(L[k]): v for k, v in p.nat_base.items()} == g["natural_base_by_length"]
    got = {f"{L[c['seq']]},{c['c']}": c["gathered_row"] for c in p.chunks}
    assert got == g["gathered_row_by_length_chunk"]


def test_toy_useful_work(golden):
    g = golden("toy_c1_plan.json")
    assert sum(causal_pairs(S) for S in g["lengths"]) == g["useful_pairs"]
    assert useful_flops(g["lengths"], 2, 64) == g["useful_fwd_bwd_flop_hq2_d64"]


def test_chunks_partition_every_sequence():
    # R20: the 2N chunks tile [0, S) exactly, including S < 2N (empty chunks)
    for S in list(range(0, 40)) + [1000, 131072]:
        for N in (1, 2, 3, 4, 8):
            edges = [chunk_bounds(S, c, N) for c in range(2 * N)]
            assert edges[0][0] == 0 and edges[-1][1] == S
            assert all(edges[i][1] == edges[i + 1][0] for i in range(2 * N - 1))
            assert sorted(chunk_owner(c, N) for c in range(2 * N)) == sorted(list(range(N)) * 2)


def test_pack_invariants_fuzz():
    rng = random.Random(3)
    m = Model(896, 128)
    for _ in range(200):
        N = rng.choice([1, 2, 4, 8])
        K = rng.randint(1, 30)
        L = [rng.randint(1, 3000) for _ in range(K)]
        C = rng.randint(max(max(L) // N + 1, -(-sum(L) // N)), sum(L) // N + 1000)
        A = dacp(L, C, N, m).assign
        p = pack_microbatch(L, A, N)
        total = 0
        for j, r in enumerate(p.ranks):
            n = r.cu_seqlens_q[-1]
            total += n
            assert sorted(r.src_row) == list(range(n))            # a permutation
            assert r.dist_rows == r.cu_seqlens_q[r.n_dist_seg]    # distributed prefix (R21)
            for i in range(len(r.q_pos)):
                ql = r.cu_seqlens_q[i + 1] - r.cu_seqlens_q[i]
                assert r.k_len[i] == r.q_pos[i] + ql               # bottom-right causal (R23)
        assert total == sum(L)
        assert p.pad_rows == max(r.dist_rows for r in p.ranks)
        assert p.natural_rows == sum(L[k] for k in range(K) if A[k] == -1)
        # gathered rows point inside the owner's padded slot (R22)
        for c in p.chunks:
            assert c["owner"] * p.pad_rows <= c["gathered_row"]
            assert c["gathered_row"] + c["len"] <= (c["owner"] + 1) * p.pad_rows
        # zigzag balances causal pairs of each distributed sequence (Eq. 4)
        for k in range(K):
            if A[k] == -1 and L[k] >= 64 * N:
                pr = rank_pairs([L[k]], [-1], N)
                assert max(pr) / (sum(pr) / N) < 1.1


def test_plan_floor():
    # all-local balanced -> 1; one long local on rank 0 of 2 -> 2
    assert plan_floor([([10, 10], [0, 1])], 2) == 1.0
    assert plan_floor([([10], [0])], 2) == 2.0
    assert abs(plan_floor([([1000], [-1])], 2) - 1.0) < 1e-3
