"""compute-sanitizer target: toy C1 (BASELINE configs[0]) at CP = 2 through the CP
runtime with the loopback exchange, in bf16 (tcgen05 kernels) and in fp32 test mode, plus the
composite skr_cp_attn_fwd / _bwd step on a 1-rank NCCL communicator with hand-distributed
sequences, the query-banded backward work lists (band_rows = 128) and the ring-CP exchange. Small on purpose: every launch runs under the sanitizer's instrumentation.

    compute-sanitizer --tool memcheck python profiles/sanitize_c1.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_19609_b200 import skrull as sk  # noqa: E402
from paper_2505_19609_b200.runtime import (RankStep, gather_rank_natural, loopback_ring_step,  # noqa: E402
                                           loopback_step)
from synth import seq_tensors  # noqa: E402

LENS = [17, 33, 64, 90, 128, 200, 256, 300]


def run(dtype, hq, hkv, d, N=2, C=600, band=None, ring=False):
    shape = sk.attn_shape(hq, hkv, d, dtype)
    p = sk.skr_plan(LENS, C, N, 1, hq * d, hkv * d)
    tdt = torch.bfloat16 if dtype == sk.SKR_BF16 else torch.float32
    inputs = [seq_tensors(0, i, S, hq, hkv, d, bf16=dtype == sk.SKR_BF16) for i, S in enumerate(LENS)]
    ranks = [RankStep(shape, np.asarray(LENS), p["assign"], N, r, band_rows=band, ring=ring) for r in range(N)]
    srcs = {k: [torch.from_numpy(gather_rank_natural(inputs, LENS, p["assign"], N, r, k)).to("cuda", tdt)
                for r in range(N)] for k in ("q", "k", "v", "do")}
    (loopback_ring_step if ring else loopback_step)(ranks, srcs["q"], srcs["k"], srcs["v"], srcs["do"])
    torch.cuda.synchronize()
    return ranks


def run_nccl():
    shape = sk.attn_shape(4, 2, 128, sk.SKR_BF16)
    lens, assign = [300, 17, 129, 64], [-1, 0, -1, 0]
    inputs = [seq_tensors(1, i, S, 4, 2, 128) for i, S in enumerate(lens)]
    rs = RankStep(shape, np.asarray(lens), np.asarray(assign, np.int32), 1, 0)
    src = {k: torch.from_numpy(gather_rank_natural(inputs, lens, assign, 1, 0, k)).to("cuda", torch.bfloat16)
           for k in ("q", "k", "v", "do")}
    comm = sk.Comm(1, 0)
    side = torch.cuda.Stream()
    rs.forward(src["q"], src["k"], src["v"], comm, side)
    rs.backward(src["do"], comm, side)
    comm.wait(torch.cuda.current_stream(), 120.0)
    comm.close()


if __name__ == "__main__":
    run(sk.SKR_BF16, 2, 2, 64)
    run(sk.SKR_BF16, 2, 1, 64)
    run(sk.SKR_BF16, 4, 2, 128)
    run(sk.SKR_FP32, 2, 2, 64)
    run(sk.SKR_BF16, 4, 2, 128, band=128)   # query-banded backward items (band accumulators, zero / cast)
    run(sk.SKR_FP32, 2, 2, 64, band=128)
    run(sk.SKR_BF16, 4, 2, 128, ring=True)   # row f4's ring CP (partials, merge, accumulate-mode backward)
    run(sk.SKR_FP32, 2, 2, 64, ring=True)
    run_nccl()
    print("sanitize target done")
