"""GPU: bench.py's multi-rank flow (torchrun, DP x CP grid, the row f3 peer exchange, max-over-ranks
timing, one JSON line from rank 0) run end to end with 2 ranks sharing ONE GPU: control plane over
gloo (SKR_BENCH_BACKEND=gloo), data plane over CUDA IPC. The numbers are meaningless (two ranks
time-share one GPU); the test checks that the multi-rank path runs and reports consistently."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("extra,cp,dp", [(["--exchange", "peer"], 2, 1), (["--dp", "2"], 1, 2),
                                         # the default workload at N = 2 (S4n2: the 128K sequence sharded)
                                         (["--exchange", "peer", "--config", "S4n2"], 2, 1)])
def test_bench_two_ranks_one_gpu(extra, cp, dp):
    env = dict(os.environ, SKR_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
           "--warmup", "1", "--no-cpu-baseline", "--no-e2e", "--config", "C2"] + extra
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["config"]["cp"] == cp and j["config"]["dp"] == dp
    assert j["value"] > 0 and j["max_mean_rank_time"] >= 1.0 and j["gpu_launches"] > 0
    if j["config"]["workload"] == "S4n2":
        assert j["config"]["distributed_seqs"] >= 1 and j["scaling"] == "strong"
