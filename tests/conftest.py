import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture
def golden():
    import json

    def load(name):
        with open(os.path.join(GOLDEN, name)) as f:
            return json.load(f)
    return load


def pytest_terminal_summary(terminalreporter):
    """Parity figures of every oracle comparison made through tests/attn_harness.tol_ok: the plain
    max-abs error per tensor kind, how many elements exceed the north_star's 2e-2 (the R34'
    bound adds the bf16 half-ulp on top of it) and how many needed R34''s operand-rounding term
    (DESIGN.md §9)."""
    h = sys.modules.get("tests.attn_harness")
    if h is None or not h.STATS:
        return
    import json
    agg = {}
    for label, kind, mx, above, n, beyond in h.STATS:
        key = (kind, label.split(" ")[0] if label else "?")
        a = agg.setdefault(key, [0.0, 0, 0, 0, 0])
        a[0] = max(a[0], mx)
        a[1] += above
        a[2] += n
        a[3] += 1
        a[4] += beyond
    tr = terminalreporter
    tr.write_sep("-", "parity vs the fp64 oracle (plain max-abs; elements > 2e-2)")
    for (kind, t), (mx, above, n, c, beyond) in sorted(agg.items()):
        tr.write_line(f"{kind} {t:6s}: {c:5d} comparisons, {n:12d} elements, max-abs {mx:.3e}, "
                      f"> 2e-2: {above} ({above / max(n, 1):.2e}), beyond R34' (within R34''): {beyond}")
    out = os.environ.get("SKR_PARITY_LOG")
    if out:
        with open(out, "w") as f:
            json.dump([{"label": l, "kind": k, "max_abs": m, "n_above_2e-2": a, "n": n, "n_beyond_r34p": b}
                       for l, k, m, a, n, b in h.STATS], f)
