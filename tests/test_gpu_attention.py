"""GPU parity: the CUDA attention path (C-ABI) vs the fp64 oracle, element by element.

Sizes span several 128-row tiles, ragged tails, empty / 1-token segments and offset query
chunks (distributed zigzag segments, R20-R23).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.attn_harness import Packed, local_pack, make_inputs, oracle_seq, tol_ok  # noqa: E402


def _sk():
    from paper_2505_19609_b200 import skrull
    return skrull


def _run_fwd(sk, shape, pk, dtype):
    segs = sk.make_segs(shape, pk.cu, pk.q_pos, pk.k_start, pk.k_len, "fwd")
    o = torch.zeros_like(pk.q)
    lse = torch.zeros(shape.hq, max(pk.rows, 1), device="cuda", dtype=torch.float32)
    sk.skr_attn_fwd(shape, segs, pk.q, pk.k, pk.v, o, lse)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), lse.cpu().numpy()


def _check_fwd(pk, O, LSE, fp32):
    r = 0
    for (s, lo, hi), in zip(((x,) for x in pk.segs)):
        Oref, Lref, *_ = oracle_seq(pk.inputs[s], bwd=False)
        n = hi - lo
        ok, err, bound = tol_ok(O[r:r + n], Oref[lo:hi], fp32)
        assert ok, f"O seq {s} [{lo},{hi}): err {err} > {bound}"
        lerr = np.abs(LSE[:, r:r + n] - Lref[:, lo:hi]).max() if n else 0.0
        assert lerr <= (1e-5 * max(1, np.abs(Lref).max()) if fp32 else 2e-2), f"LSE seq {s}: {lerr}"
        r += n


SHAPES = [(14, 2, 64), (8, 2, 128), (4, 4, 64), (3, 1, 128)]


@pytest.mark.parametrize("hq,hkv,d", SHAPES)
def test_fwd_bf16_local_ragged(hq, hkv, d):
    sk = _sk()
    lens = [1, 17, 128, 129, 300, 777, 0, 256, 1100]
    inputs = make_inputs(lens, hq, hkv, d, seed=1)
    pk = local_pack(inputs, torch.bfloat16)
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
    O, L = _run_fwd(sk, shape, pk, torch.bfloat16)
    _check_fwd(pk, O, L, fp32=False)


@pytest.mark.parametrize("hq,hkv,d", SHAPES[:2])
def test_fwd_bf16_peaky_softmax(hq, hkv, d):
    # sigma 3 Q/K: large logits exercise the lazy O rescale
    sk = _sk()
    lens = [700, 1500]
    inputs = make_inputs(lens, hq, hkv, d, seed=2, sigma_qk=3.0)
    pk = local_pack(inputs, torch.bfloat16)
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16)
    O, L = _run_fwd(sk, shape, pk, torch.bfloat16)
    _check_fwd(pk, O, L, fp32=False)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("N", [1, 2, 4])
def test_fwd_distributed_chunks(dtype, N):
    # one rank's zigzag chunks (R20) of three sequences against their natural K/V buffers
    sk = _sk()
    hq, hkv, d = 8, 2, 64
    lens = [5, 700, 1333]
    bf = dtype == "bf16"
    inputs = make_inputs(lens, hq, hkv, d, seed=3, bf16=bf)
    tdt = torch.bfloat16 if bf else torch.float32
    shape = sk.attn_shape(hq, hkv, d, sk.SKR_BF16 if bf else sk.SKR_FP32)
    base, acc = {}, 0
    for s, S in enumerate(lens):
        base[s] = acc
        acc += S
    for j in range(N):
        segs = []
        for s, S in enumerate(lens):
            for c in (j, 2 * N - 1 - j):
                segs.append((s, c * S // (2 * N), (c + 1) * S // (2 * N)))
        pk = Packed(inputs, segs, base, list(range(len(lens))), tdt)
        O, L = _run_fwd(sk, shape, pk, tdt)
        _check_fwd(pk, O, L, fp32=not bf)


def test_fwd_fp32_local():
    sk = _sk()
    lens = [1, 33, 64, 90, 200, 300]
    inputs = make_inputs(lens, 2, 2, 64, seed=4, bf16=False)
    pk = local_pack(inputs, torch.float32)
    shape = sk.attn_shape(2, 2, 64, sk.SKR_FP32)
    O, L = _run_fwd(sk, shape, pk, torch.float32)
    _check_fwd(pk, O, L, fp32=True)
