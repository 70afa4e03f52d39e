"""GPU parity of the opt-in CTA-pair (cta_group::2) d = 128 forward (SKR_FWD_2SM=1).

The mode is read once per process (it also switches skr_attn_block_m to 256-row super tiles), so
the d = 128 attention parity tests run again in a child process with the variable set: same
inputs, same oracle, same tolerances as tests/test_gpu_attention.py (forward, and the backward
that consumes its O / LSE)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_fwd_cta_pair_parity():
    env = dict(os.environ, SKR_FWD_2SM="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gpu_attention.py", "-k", "128"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


def test_block_m_switches_to_super_tiles():   # host logic, no GPU
    code = ("from paper_2505_19609_b200 import skrull as sk;"
            "print(sk.skr_attn_block_m(sk.attn_shape(8, 2, 128, sk.SKR_BF16)),"
            " sk.skr_attn_block_m(sk.attn_shape(8, 2, 64, sk.SKR_BF16)))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, SKR_FWD_2SM="1"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.split() == ["256", "128"]
