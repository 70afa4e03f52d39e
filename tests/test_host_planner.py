"""C-ABI host planner (libskrull.so) vs the independent oracle: bit-exact plans and tables.

No GPU needed: these call only host entry points of the library.
"""
import os
import random
import re
from fractions import Fraction

import numpy as np
import pytest

from oracle.cost_model import Fit, Model, flops, volume
from oracle.pack import pack_microbatch
from oracle.schedule import GDSError, ScheduleError, dacp, eval_tdacp, gds, lpt, plan

skrull = pytest.importorskip("paper_2505_19609_b200.skrull")

SHAPES = [(896, 128), (3584, 512), (4096, 1024), (64, 16), (1, 1)]


def test_abi_exports_every_declared_symbol():
    declared = skrull._declared_names()
    assert len(declared) > 30
    missing = [n for n in declared if n not in skrull.exported_symbols()]
    assert not missing, missing
    assert skrull.skr_abi_version() >= 1


def test_cost_model_matches_oracle():
    for h, hkv in SHAPES:
        for S in (0, 1, 17, 4096, 131072, 1_643_000):
            assert skrull.skr_flops(S, h, hkv) == flops(S, Model(h, hkv))
            assert skrull.skr_volume(S, h, hkv) == volume(S, Model(h, hkv))
    with pytest.raises(skrull.SkrullError) as e:
        skrull.skr_flops(2 ** 40, 4096, 1024)
    assert e.value.status == skrull.SKR_E_OVERFLOW
    assert skrull.skr_t_comp(0, 3, 9) == 0 and skrull.skr_t_comp(1000, 0.5, 10) == 510
    assert skrull.skr_t_comm(0, 3, 9) == 0 and skrull.skr_t_comm(4, 1, 0) == 4
    s, i = skrull.skr_fit_linear([1, 2, 3, 4], [7, 9, 11, 13])
    assert abs(s - 2) < 1e-12 and abs(i - 5) < 1e-12
    with pytest.raises(skrull.SkrullError):
        skrull.skr_fit_linear([2], [80.62])
    assert skrull.skr_bucket_size(210, 2, 10) == 100
    with pytest.raises(skrull.SkrullError):
        skrull.skr_bucket_size(10, 2, 10)


def _lens(rng, K, mu=5.0, sigma=1.3, hi=20000):
    return [int(min(hi, max(1, round(rng.lognormvariate(mu, sigma))))) for _ in range(K)]


def test_dacp_bit_exact_fuzz():
    rng = random.Random(11)
    n_err = 0
    for it in range(1500):
        N = rng.choice([1, 2, 3, 4, 8])
        K = rng.randint(0, 60)
        h, hkv = rng.choice(SHAPES)
        L = _lens(rng, K)
        tot = sum(L)
        C = rng.randint(max(1, (max(L) if L else 1) // N // 2), max(2, tot // N + 500))
        rb = rng.random() < 0.85
        try:
            ref = dacp(L, C, N, Model(h, hkv), rb)
        except ScheduleError as e:
            n_err += 1
            with pytest.raises(skrull.SkrullError) as ce:
                skrull.skr_dacp(L, C, N, h, hkv, rollback=rb)
            assert ce.value.status == skrull.SKR_E_SCHEDULE
            assert ce.value.fail_idx == e.pos
            continue
        A, nrb = skrull.skr_dacp(L, C, N, h, hkv, rollback=rb)
        assert list(A) == ref.assign, (L, C, N)
        assert nrb == ref.n_rollbacks
    assert 50 < n_err < 1400


def test_eval_tdacp_matches_oracle():
    rng = random.Random(12)
    for _ in range(300):
        N = rng.choice([1, 2, 4])
        K = rng.randint(1, 12)
        L = _lens(rng, K, hi=5000)
        A = [rng.randint(-1, N - 1) for _ in range(K)]
        C = rng.randint(1, 6000)
        comp, comm = (1e-9, 3.0), (2e-6, 100.0)
        r = skrull.skr_eval_tdacp(L, A, C, N, 896, 128, comp, comm, bytes_per_elem=2, dist_penalty=1.2)
        o = eval_tdacp(L, A, C, N, Model(896, 128), Fit(*comp), Fit(*comm), 2, Fraction(6, 5))
        assert r["feasible"] == o.feasible
        assert abs(r["tdacp"] - float(o.tdacp)) <= 1e-9 * max(1.0, float(o.tdacp))
        assert abs(r["comm_time"] - float(o.comm_time)) <= 1e-9 * max(1.0, float(o.comm_time))
        np.testing.assert_allclose(r["per_rank_time"], [float(x) for x in o.per_rank_time], rtol=1e-9)


def test_worked_tdacp_examples():
    # 144 / 160 / 84 under identity fits, h = h_kv = b = 1
    assert skrull.skr_eval_tdacp([4, 2, 2], [-1, 0, 1], 100, 2, 1, 1, (1, 0), (1, 0))["tdacp"] == 144
    assert skrull.skr_eval_tdacp([4], [0], 100, 2, 1, 1, (1, 0), (1, 0))["tdacp"] == 160
    assert skrull.skr_eval_tdacp([4], [-1], 100, 2, 1, 1, (1, 0), (1, 0))["tdacp"] == 84


def test_lpt_gds_plan_bit_exact_fuzz():
    rng = random.Random(13)
    for _ in range(300):
        N = rng.choice([1, 2, 4, 8])
        ws = rng.choice([1, 2, 4])
        K = rng.randint(1, 80)
        h, hkv = rng.choice(SHAPES[:3])
        L = _lens(rng, K)
        C = rng.randint(max(1, max(L) // (2 * N)), max(L) + 4000)
        m = Model(h, hkv)
        assert list(skrull.skr_lpt(L, ws, h, hkv)) == lpt(L, ws, m)
        try:
            ref = plan(L, C, N, ws, m)
        except (GDSError, ScheduleError):
            with pytest.raises(skrull.SkrullError):
                skrull.skr_plan(L, C, N, ws, h, hkv)
            continue
        p = skrull.skr_plan(L, C, N, ws, h, hkv)
        assert list(p["dp_of_seq"]) == ref.dp_of_seq
        assert list(p["mb_of_seq"]) == ref.mb_of_seq
        assert list(p["assign"]) == ref.assign
        assert list(p["n_mb_per_dp"]) == ref.n_mb
        assert p["n_rollbacks"] == ref.n_rollbacks
        for i in range(ws):
            mbo, n = skrull.skr_gds(L, C, N, ws, i, h, hkv)
            assert n == ref.n_mb[i]


def test_toy_plan_through_abi(golden):
    g = golden("toy_c1_plan.json")
    p = skrull.skr_plan(g["lengths"], g["C"], g["N"], 1, g["hidden"], g["kv_hidden"])
    assert list(p["assign"]) == g["assign"] and p["n_rollbacks"] == g["n_rollbacks"]
    assert list(p["n_mb_per_dp"]) == [g["gds_init"]]
    for j, key in enumerate(("rank0", "rank1")):
        r = skrull.skr_pack_rank(g["lengths"], g["assign"], g["N"], j)
        assert list(r["cu_seqlens_q"]) == g[key]["cu_seqlens_q"]
        assert list(r["q_pos"]) == g[key]["q_pos"]
        assert list(r["k_len"]) == g[key]["k_len"]
        assert r["pad_rows_P"] == g["pad_rows_P"] and r["natural_rows"] == g["natural_rows"]


def test_pack_bit_exact_fuzz():
    rng = random.Random(14)
    for _ in range(300):
        N = rng.choice([1, 2, 3, 4, 8])
        K = rng.randint(0, 40)
        L = [rng.randint(0, 3000) for _ in range(K)]
        A = [rng.randint(-1, N - 1) for _ in range(K)]
        ref = pack_microbatch(L, A, N)
        t = skrull.skr_pack_chunks(L, A, N)
        assert len(t) == len(ref.chunks)
        for row, c in zip(t, ref.chunks):
            assert list(row) == [c["seq"], c["c"], c["owner"], c["gathered_row"], c["natural_row"], c["len"]]
        for j in range(N):
            r = skrull.skr_pack_rank(L, A, N, j)
            o = ref.ranks[j]
            assert list(r["cu_seqlens_q"]) == o.cu_seqlens_q
            assert list(r["q_pos"]) == o.q_pos
            assert list(r["k_start"]) == o.k_start
            assert list(r["k_len"]) == o.k_len
            assert list(r["seg_seq"]) == o.seg_seq
            assert list(r["seg_chunk"]) == o.seg_chunk
            assert list(r["src_row"]) == o.src_row
            assert r["dist_rows"] == o.dist_rows and r["pad_rows_P"] == ref.pad_rows
            assert r["n_dist_seg"] == o.n_dist_seg


def test_owner_row_map(golden):
    # row f3 step two: natural distributed row -> owner * P + prefix row. Pinned to the hand-traced
    # toy C1 gathered rows and, by fuzz, to the oracle packer's chunk table: each
    # chunk's rows map to consecutive rows of its owner's prefix, and every owner prefix row of a
    # distributed sequence is hit exactly once.
    L, A = [17, 33, 64, 90, 128, 200, 256, 300], [-1, 1, -1, 1, 0, 1, 0, -1]
    m = skrull.skr_pack_owner_rows(skrull.skr_pack_chunks(L, A, 2), 381)
    P = 191
    # 17c0 -> 0, 17c1 -> 191, 17c2 -> 195, 17c3 -> 4; 64c0 -> 9; 300c3 -> 116 (natural base 81 + 225)
    assert list(m[0:17]) == [0, 1, 2, 3, 191, 192, 193, 194, 195, 196, 197, 198, 4, 5, 6, 7, 8]
    assert m[17] == 9 and m[81 + 225] == 116 and m[81 + 75] == 231
    rng = random.Random(41)
    for _ in range(200):
        N = rng.choice([1, 2, 3, 4, 8])
        K = rng.randint(0, 30)
        L = [rng.randint(0, 2000) for _ in range(K)]
        A = [rng.randint(-1, N - 1) for _ in range(K)]
        ref = pack_microbatch(L, A, N)
        nat = sum(S for S, a in zip(L, A) if a == -1)
        m = skrull.skr_pack_owner_rows(skrull.skr_pack_chunks(L, A, N), nat)
        want = np.full(nat, -1)
        for c in ref.chunks:
            want[c["natural_row"]:c["natural_row"] + c["len"]] = c["gathered_row"] + np.arange(c["len"])
        assert np.array_equal(m, want)
        P = ref.pad_rows
        if P:
            owners, rows = m // P, m % P
            for j in range(N):
                mine = np.sort(rows[owners == j])
                assert np.array_equal(mine, np.arange(ref.ranks[j].dist_rows))
    with pytest.raises(skrull.SkrullError):
        skrull.skr_pack_owner_rows(skrull.skr_pack_chunks([10], [-1], 2), 9)   # table exceeds the rows


def test_tiles_cover_work_once_and_are_lpt_ordered():
    rng = random.Random(15)
    for _ in range(50):
        n = rng.randint(0, 20)
        ql = [rng.randint(0, 700) for _ in range(n)]
        qp = [rng.randint(0, 500) for _ in range(n)]
        cu = np.concatenate([[0], np.cumsum(ql)]).astype(np.int32)
        kl = [a + b for a, b in zip(qp, ql)]
        tf = skrull.skr_tiles_fwd(cu, qp, n, 128)
        assert sorted(map(tuple, tf)) == sorted((s, t) for s in range(n) for t in range(-(-ql[s] // 128)))
        w = [qp[s] + min(ql[s], (t + 1) * 128) for s, t in tf]
        assert w == sorted(w, reverse=True)
        tb = skrull.skr_tiles_bwd(cu, qp, kl, n, 128)
        assert sorted(map(tuple, tb)) == sorted((s, t, 0, ql[s]) for s in range(n) if ql[s] > 0
                                                for t in range(-(-kl[s] // 128)))
        w = [ql[s] - max(0, t * 128 - qp[s]) for s, t, _, _ in tb]
        assert w == sorted(w, reverse=True)


def test_tiles_bwd_query_bands_cover_every_causal_pair_once():
    # skr_tiles_bwd with band_rows: every (segment, key tile, visible query) exactly once; segments of
    # more than band_rows queries come first, split into bands [b*B, (b+1)*B) in (segment, band, key
    # tile) order, the rest whole and LPT-ordered after them
    rng = random.Random(17)
    for it in range(60):
        n = rng.randint(0, 8)
        ql = [rng.choice([0, 1, 127, 128, 129, 300, 700, 1024, 1500, 2500]) for _ in range(n)]
        qp = [rng.choice([0, 0, 5, 128, 333]) for _ in range(n)]
        cu = np.concatenate([[0], np.cumsum(ql)]).astype(np.int32)
        kl = [a + b for a, b in zip(qp, ql)]
        B = rng.choice([128, 256, 512, 1024])
        bn = rng.choice([32, 128])
        tb = skrull.skr_tiles_bwd(cu, qp, kl, n, bn, B)
        seen = {}
        for s, t, lo, hi in tb:
            first = max(0, t * bn - qp[s])
            assert 0 <= lo < hi <= ql[s] and max(lo, first) < hi
            for i in range(max(lo, first), hi):
                key = (s, t, i)
                assert key not in seen
                seen[key] = 1
        want = {(s, t, i) for s in range(n) for t in range(-(-kl[s] // bn))
                for i in range(max(0, t * bn - qp[s]), ql[s])}
        assert set(seen) == want
        split = [ql[s] > B for s, _, _, _ in tb]
        assert split == sorted(split, reverse=True)          # banded items first
        nb = sum(split)
        order = [(s, lo, t) for s, t, lo, _ in tb[:nb]]
        assert order == sorted(order)
        assert all(lo % B == 0 and (hi == ql[s] or hi - lo == B) for s, _, lo, hi in tb[:nb])
        assert all(lo == 0 and hi == ql[s] for s, _, lo, hi in tb[nb:])
    with pytest.raises(skrull.SkrullError):
        skrull.skr_tiles_bwd(np.array([0, 10], np.int32), [0], [10], 1, 128, 100)   # not a multiple of 128


def test_baselines_bit_exact_fuzz():
    # row f1: Alg. 4 round-robin and full-shard vs the oracle
    from oracle.schedule import full_shard, round_robin
    rng = random.Random(16)
    for _ in range(800):
        N = rng.choice([1, 2, 4, 8])
        K = rng.randint(0, 50)
        L = _lens(rng, K)
        C = rng.randint(1, max(2, sum(L) // N + 1000))
        rb = rng.random() < 0.8
        try:
            ref = round_robin(L, C, N, rb)
        except ScheduleError as e:
            with pytest.raises(skrull.SkrullError) as ce:
                skrull.skr_round_robin(L, C, N, rb)
            assert ce.value.fail_idx == e.pos
            continue
        A, _ = skrull.skr_round_robin(L, C, N, rb)
        assert list(A) == ref
        try:
            mbs = full_shard(L, C, N)
        except ScheduleError:
            with pytest.raises(skrull.SkrullError):
                skrull.skr_full_shard(L, C, N)
            continue
        M, n = skrull.skr_full_shard(L, C, N)
        assert n == len(mbs)
        assert all(M[k] == j for j, mb in enumerate(mbs) for k in mb)
    # Table 3 structure: both heuristics fail without roll-back on [50,60,90], C=100, N=2
    with pytest.raises(skrull.SkrullError):
        skrull.skr_round_robin([50, 60, 90], 100, 2, rollback=False)
    assert list(skrull.skr_round_robin([50, 60, 90], 100, 2)[0]).count(-1) >= 1


def test_header_is_plain_c_and_links(tmp_path):
    # the boundary is a C ABI: include/skrull.h compiles as strict C99 and a plain C program links
    # against libskrull.so and calls through it (host planner entry points need no GPU)
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    from paper_2505_19609_b200 import skrull
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = tmp_path / "abi.c"
    src.write_text('#include "skrull.h"\n#include <stdio.h>\n'
                   'int main(void) {\n'
                   '  skr_model m = {64, 16, 1}; int64_t f = 0;\n'
                   '  if (skr_flops(128, &m, &f) != SKR_OK) return 1;\n'
                   '  printf("%d %lld\\n", (int)skr_abi_version(), (long long)f);\n'
                   '  return 0;\n}\n')
    lib_dir = os.path.dirname(skrull.LIB_PATH)
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", os.path.join(root, "include"),
                    str(src), "-L", lib_dir, "-l:" + os.path.basename(skrull.LIB_PATH), "-Wl,-rpath," + lib_dir,
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    assert int(out[0]) == skrull.skr_abi_version() and int(out[1]) == 15204352


def test_ring_segments_visit_every_causal_key_chunk_once():
    # row f4 (ring CP): over the N hops and both key-chunk classes, every own query chunk c of every
    # distributed sequence sees each non-empty key chunk c' <= c exactly once -- whole when c' < c
    # (q_pos = its length), the causal diagonal when c' == c -- at the rows that chunk occupies in
    # the visiting rank's packed prefix (skr_pack_chunks), and nothing after c
    rng = random.Random(18)
    for it in range(120):
        N = rng.randint(1, 5)
        K = rng.randint(1, 7)
        lens = [rng.choice([1, 2, 3, 7, 64, 129, 300, 1000]) for _ in range(K)]
        assign = [-1 if rng.random() < 0.5 else rng.randrange(N) for _ in range(K)]
        table = skrull.skr_pack_chunks(lens, assign, N)
        P = skrull.skr_pack_bounds(lens, assign, N, 0)["pad_rows_P"]
        where = {(int(t[0]), int(t[1])): (int(t[3]) - int(t[2]) * P, int(t[5])) for t in table}
        dist = [k for k in sorted(range(K), key=lambda k: (lens[k], k)) if assign[k] == -1]
        for j in range(N):
            pr = skrull.skr_pack_rank(lens, assign, N, j)
            nd = 2 * len(dist)
            seen = {}
            for r in range(N):
                s = (j - r) % N
                for cls in (0, 1):
                    t = skrull.skr_ring_segs(lens, assign, N, j, r, cls)
                    assert t["n_seg"] == nd
                    assert list(t["cu_seqlens_q"]) == list(pr["cu_seqlens_q"][:nd + 1])
                    ck = s if cls == 0 else 2 * N - 1 - s
                    for i in range(nd):
                        k, c = dist[i // 2], (j, 2 * N - 1 - j)[i % 2]
                        if t["k_len"][i] == 0:
                            assert ck > c or where[(k, ck)][1] == 0
                            continue
                        off, ln = where[(k, ck)]
                        assert ck <= c and t["k_start"][i] == off and t["k_len"][i] == ln
                        assert t["q_pos"][i] == (ln if ck < c else 0)
                        assert (k, c, ck) not in seen
                        seen[(k, c, ck)] = 1
            want = {(k, c, cc) for k in dist for c in (j, 2 * N - 1 - j) for cc in range(c + 1)
                    if where[(k, cc)][1] > 0}
            assert set(seen) == want
