"""Input generators: calibration to PAPER.md Table 1 and determinism."""
import numpy as np

from synth import CONFIGS, gen_lengths, quantiles, seq_tensors, round_bf16


def test_longtail_matches_wikipedia_row(golden):
    t = golden("table1_quantiles.json")
    fr, _ = quantiles(gen_lengths("longtail", 100_000, 7), t["thresholds"][:3])
    for got, want in zip(fr, t["Wikipedia"][:3]):
        assert abs(got - want) <= 0.03


def test_bimodal_matches_chatqa2_row(golden):
    t = golden("table1_quantiles.json")
    fr, longest = quantiles(gen_lengths("bimodal", 100_000, 7), t["thresholds"][:4])
    assert abs(fr[2] - t["ChatQA2-Long-SFT"][2]) <= 0.05            # <8K within 5 pts
    assert abs(fr[0] - t["ChatQA2-Long-SFT"][0]) <= 0.05
    assert longest <= 32768


def test_short1k_is_llama3_like():
    # 99.89 % short (< 1K)
    x = gen_lengths("short1k", 10_000, 0)
    assert x.max() <= 1023 and x.min() >= 16


def test_determinism_and_configs():
    assert np.array_equal(gen_lengths("longtail", 50, 3), gen_lengths("longtail", 50, 3))
    c2 = CONFIGS["C2"].lengths(0)
    assert len(c2) == 64 and c2[-1] == 32768 and c2.max() <= 32768
    c4 = CONFIGS["C4"].lengths(0)
    assert len(c4) == 512 and (c4 < 1024).mean() > 0.99
    a = seq_tensors(0, 3, 10, 4, 2, 8)
    b = seq_tensors(0, 3, 10, 4, 2, 8)
    assert all(np.array_equal(a[n], b[n]) for n in a)


def test_round_bf16():
    x = np.array([1.0, 1.00390625, 1.0078125, 1.01171875, -3.3e-3, 65504.0], np.float32)
    r = round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.0078125 and r[3] == 1.015625  # RNE ties
    assert np.all((r.view(np.uint32) & 0xFFFF) == 0)
