"""GPU: UMMA / TMA / TMEM building blocks through every operand layout the kernels use."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [64, 128])
@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_umma_layouts(variant, n):
    from paper_2505_19609_b200 import skrull
    g = torch.Generator(device="cuda").manual_seed(variant * 7 + n)
    A = torch.randn(128, 128, device="cuda", generator=g).bfloat16()
    if variant in (1, 2):
        B = torch.randn(128, n, device="cuda", generator=g).bfloat16()   # [K][n]
    else:
        B = torch.randn(n, 128, device="cuda", generator=g).bfloat16()   # [n][K]
    C = torch.zeros(128, n, device="cuda")
    skrull.skr_selftest_umma(variant, n, A, B, C)
    torch.cuda.synchronize()
    Af, Bf = A.float(), B.float()
    if variant in (0, 3, 4):
        ref = Af @ Bf.T
    elif variant == 1:
        ref = Af @ Bf
    else:
        ref = Af.T @ Bf            # A given as [K][M]
    err = (C - ref).abs().max().item()
    assert err < 1e-2 * max(1.0, ref.abs().max().item()), err
