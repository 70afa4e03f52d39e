"""GPU parity of the CTA-pair (cta_group::2) d = 128 forward, the libskrull_fwd2sm.so build variant.

The variant is a separate library (its skr_attn_block_m answers 256-row super tiles for d = 128),
so the d = 128 attention parity tests run again in a child process that loads it through
SKR_LIB_PATH: same inputs, same oracle, same tolerances as tests/test_gpu_attention.py (forward,
and the backward that consumes its O / LSE)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANT_LIB = os.path.join(ROOT, "paper_2505_19609_b200", "libskrull_fwd2sm.so")


def _env():
    if not os.path.exists(VARIANT_LIB):
        pytest.skip("libskrull_fwd2sm.so not built (__graft_entry__.build() builds it)")
    return dict(os.environ, SKR_LIB_PATH=VARIANT_LIB)


@pytest.mark.gpu
def test_fwd_cta_pair_parity():
    env = _env()
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "tests/test_gpu_attention.py", "-k", "128"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


def test_block_m_switches_to_super_tiles():   # host logic, no GPU: fixed per library build
    code = ("from paper_2505_19609_b200 import skrull as sk;"
            "print(sk.skr_attn_block_m(sk.attn_shape(8, 2, 128, sk.SKR_BF16)),"
            " sk.skr_attn_block_m(sk.attn_shape(8, 2, 64, sk.SKR_BF16)))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=_env(),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.split() == ["256", "128"]


def test_production_block_m_ignores_environment():   # host logic, no GPU
    code = ("from paper_2505_19609_b200 import skrull as sk;"
            "print(sk.skr_attn_block_m(sk.attn_shape(8, 2, 128, sk.SKR_BF16)))")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=dict(os.environ, SKR_FWD_2SM="1"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.split() == ["128"]
