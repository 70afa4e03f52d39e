"""Row f2: the cost model calibrated on B200 (tools/calibrate.py ->
profiles/r01_calibration.json) and the DACP heuristic compared with the exhaustive optimum in real
seconds under it (S:278, S:469, S:561 asked for this comparison under measured fits).

The calibration numbers are measurements, not paper values: they are "parity unpinned" (DESIGN.md
§4). What is checked here is (a) that the committed measurement is internally consistent (fits
reproduce their points, the Fig. 1b analog has the shape PAPER.md P:75-80 describes for short
sequences), and (b) that the heuristic never beats the optimum and stays close to it under FIT_B200.
"""
import json
import os
import random

import pytest

from oracle.cost_model import Fit, Model
from oracle.schedule import ScheduleError, dacp, eval_tdacp, optimal_dacp

CAL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "r01_calibration.json")
QWEN7 = Model(3584, 512, 1)
# Table 5 all_gather fit (SURVEY §8(c) FIT_B200 comm until a multi-GPU sweep exists):
# 6.256 us/MB + 116.5 us, Volume in elements x 2 B (R25)
TABLE5_AG = Fit(6.256e-6 / (1 << 20), 116.5e-6)


@pytest.fixture(scope="module")
def cal():
    if not os.path.exists(CAL):
        pytest.skip("no calibration committed")
    with open(CAL) as f:
        return json.load(f)


def test_comp_fit_reproduces_points(cal):
    for name, r in cal["t_comp"].items():
        f = r["fit_useful"]
        assert f["slope_s_per_flop"] > 0 and f["r2"] > 0.98, name
        # the asymptotic rate of the useful-FLOP fit is a plausible B200 attention rate
        assert 300 < f["tflops_asymptotic"] < 2250, name
        # long sequences (>= 16K) are predicted within 30 % by the fit (shorter ones run below the
        # asymptotic rate: tile quantisation and launch overhead, the Fig. 1b effect)
        for p in r["points"]:
            if p["S"] >= 16384:
                pred = f["slope_s_per_flop"] * p["useful_flops"] + f["intercept_s"]
                assert abs(pred - p["t_s"]) <= 0.3 * p["t_s"], (name, p["S"])


def test_fig1b_shape(cal):
    # P:75-80 / P:101: sharding a SHORT sequence over a CP group costs per-GPU efficiency; long
    # sequences keep it (that is why DACP keeps short sequences local)
    pts = {(p["S"], p["N"]): p["per_gpu_tflops"] for p in cal["fig1b"]["points"]}
    assert pts[(1024, 8)] < 0.5 * pts[(1024, 1)]
    assert pts[(16384, 8)] > 0.8 * pts[(16384, 1)]


def _fit_b200(cal):
    f = cal["t_comp"]["qwen7"]["fit_eq12"]
    return Fit(f["slope_s_per_flop"], f["intercept_s"])


def test_heuristic_vs_optimum_in_seconds(cal):
    comp = _fit_b200(cal)
    rng = random.Random(11)
    ratios = []
    while len(ratios) < 60:
        N = rng.choice([2, 4])
        K = rng.randint(2, 5 if N == 4 else 6)
        # Long-SFT-like: mostly short, some long
        lens = [int(min(65536, max(64, rng.lognormvariate(6.5, 1.6)))) for _ in range(K)]
        C = rng.randint(max(max(lens) // N + 1, sum(lens) // N), sum(lens) // N + 8192)
        try:
            r = dacp(lens, C, N, QWEN7)
        except ScheduleError:
            continue
        opt = optimal_dacp(lens, C, N, QWEN7, comp, TABLE5_AG, 2)
        assert opt is not None
        h = eval_tdacp(lens, r.assign, C, N, QWEN7, comp, TABLE5_AG, 2).tdacp
        assert h >= opt[1] * (1 - 1e-12)
        ratios.append(h / opt[1])
    ratios.sort()
    # measured at freeze time under the r01 B200 fit: median 1.24, p90 1.96, max 2.46 -- with
    # attention at ~0.9 PFLOP/s a forced shard's fixed all-gather cost (116.5 us, Table 5) weighs
    # more against short compute than on H100, and Alg. 1 never weighs T_comm (R25)
    assert ratios[len(ratios) // 2] <= 1.3
    assert ratios[int(0.9 * len(ratios))] <= 2.1
    assert ratios[-1] <= 2.6
