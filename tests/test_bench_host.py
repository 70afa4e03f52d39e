"""CPU: the bench's host-side arithmetic against the oracle's independent accounting (R32, the
SURVEY §8(d) plan floor), and the runtime's grid / buffer-pool bookkeeping (no GPU needed)."""
import os
import random
import sys

import numpy as np
import pytest

from oracle import metrics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def bench():
    import bench as b
    return b


def test_useful_flops_matches_oracle(bench):
    from synth.configs import QWEN05, LLAMA8
    rng = random.Random(3)
    for shp in (QWEN05, LLAMA8):
        lens = [rng.randint(1, 40000) for _ in range(37)]
        assert bench.useful_flops(lens, shp) == metrics.useful_flops(lens, shp.hq, shp.d)


def test_rank_pairs_and_plan_floor_match_oracle(bench):
    sk = pytest.importorskip("paper_2505_19609_b200.skrull")
    from paper_2505_19609_b200.runtime import dp_micro_batches
    from synth import CONFIGS
    for name, N, C in (("C2", 1, 65536), ("C2", 4, 30720), ("C5n8", 8, 65536)):
        cfg = CONFIGS[name]
        lens = np.concatenate([cfg.lengths(r) for r in range(N)]) if name == "C2" else cfg.lengths(0)
        p = sk.skr_plan(lens, C, N, 1, cfg.shape.hidden, cfg.shape.kv_hidden)
        mbs = [(ml, ma) for _, ml, ma in dp_micro_batches(p, lens, 0)]
        for ml, ma in mbs:
            assert [bench.rank_pairs(ml, ma, N, r) for r in range(N)] == metrics.rank_pairs(ml, ma, N)
        # bench's Eq. 8-style floor (DP = 1) equals the oracle's
        pp = [[bench.rank_pairs(ml, ma, N, r) for r in range(N)] for ml, ma in mbs]
        floor = sum(max(x) for x in pp) / (sum(sum(x) for x in pp) / N)
        assert abs(floor - metrics.plan_floor(mbs, N)) < 1e-12


def test_grid_coords_and_dp_micro_batches():
    sk = pytest.importorskip("paper_2505_19609_b200.skrull")
    from paper_2505_19609_b200.runtime import dp_micro_batches, grid_coords
    assert [grid_coords(r, 8, 2) for r in range(8)] == [(r // 4, r % 4, 4) for r in range(8)]
    with pytest.raises(ValueError):
        grid_coords(0, 6, 4)
    lens = np.asarray([900, 37, 700, 129, 1, 600, 64, 1000, 250, 333, 4000, 17])
    p = sk.skr_plan(lens, 2500, 2, 2, 512, 128)   # GDS needs max S <= N*C
    seen = []
    for d in range(2):
        for idx, ml, ma in dp_micro_batches(p, lens, d):
            assert np.array_equal(ml, lens[idx]) and np.array_equal(ma, p["assign"][idx])
            seen += list(idx)
    assert sorted(seen) == list(range(len(lens)))          # every sequence exactly once


def test_buffer_pool_views():
    import torch
    from paper_2505_19609_b200.runtime import BufferPool
    pool = BufferPool(device="cpu")
    a = pool.reserve("x", (10, 4), torch.float32)
    b = pool.reserve("x", (3, 5), torch.float32)
    assert a.device.type == "meta" and b.device.type == "meta"
    pool.materialize()
    assert pool.bufs["x"].numel() == 40                     # the largest request
    va, vb = pool.get("x", (10, 4), torch.float32), pool.get("x", (3, 5), torch.float32)
    assert va.shape == (10, 4) and vb.shape == (3, 5) and va.data_ptr() == vb.data_ptr()


def test_workload_grid_cp_and_default(bench):
    # a named config under --dp > 1 must plan for CP = world // dp (not world)
    from types import SimpleNamespace as NS
    a = NS(config="C5n4", dp=2, seed=0)
    name, cfg, lens, shp, cp, bucket, scaling = bench.workload(a, 8)
    assert (name, cp, cfg.cp, scaling) == ("C5n4", 4, 4, "weak")
    # the default workload is S4n{CP} at every N (BENCH and SCALE share it), strong scaling
    for world, dp, want in ((1, 1, "S4n1"), (2, 1, "S4n2"), (8, 1, "S4n8"), (8, 2, "S4n4")):
        name, cfg, lens, shp, cp, bucket, scaling = bench.workload(NS(config=None, dp=dp, seed=0), world)
        assert name == want and cp == world // dp and scaling == "strong" and len(lens) == 512
    with pytest.raises(SystemExit):
        bench.workload(NS(config="C5n4", dp=1, seed=0), 8)      # CP 8 != config's 4
    with pytest.raises(SystemExit):
        bench.workload(NS(config=None, dp=3, seed=0), 8)        # dp does not divide the world


def test_pick_peak(bench):
    peaks = {"bf16_tflops": 1629.9, "bf16_tflops_sustained": 1368.0}
    (p, k), b, s = bench.pick_peak(peaks, {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0}, 8.0)
    assert (p, k) == (1629.9, "bf16_tflops")                    # full clocks: burst
    (p, k), _, _ = bench.pick_peak(peaks, {"sm_mhz": 1410.0, "sm_max_mhz": 1965.0}, 8.0)
    assert (p, k) == (1368.0, "bf16_tflops_sustained")          # seconds at power-capped clocks
    (p, k), _, _ = bench.pick_peak(peaks, {"sm_mhz": 1410.0, "sm_max_mhz": 1965.0}, 0.2)
    assert k == "bf16_tflops"                                   # a short region is a burst
