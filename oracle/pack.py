"""Oracle: per-CP-rank packed layout of one DACP micro-batch (readings R20-R23).

Test infrastructure only (see oracle/__init__.py).

PAPER.md fixes only that distributed sequences put S/N tokens on every rank
(Eq. 4, Eq. 7), that sequences are packed without padding
 and that the CP implementation is orthogonal. The layout below
is the DESIGN.md reading:
  R20 zigzag: 2N chunks [floor(cS/2N), floor((c+1)S/2N)); rank j owns chunks j and 2N-1-j.
  R21 packed order on rank j: [distributed chunks in plan order (chunk j, then 2N-1-j)]
      ++ [local sequences on j in plan order]; "plan order" = ascending (length, index).
  R22 all-gather pad P = max over ranks of the distributed-prefix rows.
  R23 distributed K/V is addressed in a natural per-sequence buffer; bottom-right causal.
Rank-natural source order (`src_row`): the rank's own rows in input-index order, each
sequence's rows by ascending position (local: whole sequence; distributed: chunk j then
chunk 2N-1-j).
"""
from __future__ import annotations

from dataclasses import dataclass


def chunk_bounds(S: int, c: int, N: int):
    """R20: chunk c of 2N, [floor(c*S/2N), floor((c+1)*S/2N))."""
    return (c * S) // (2 * N), ((c + 1) * S) // (2 * N)


def chunk_owner(c: int, N: int) -> int:
    """R20: owner(c) = c if c < N else 2N-1-c."""
    return c if c < N else 2 * N - 1 - c


@dataclass
class RankPack:
    cu_seqlens_q: list     # [n_seg+1]
    q_pos: list            # [n_seg] absolute position of the segment's first query in its sequence
    k_start: list          # [n_seg] first K row: packed row (locals) / natural-dist row (distributed)
    k_len: list            # [n_seg] keys visible to the last query (= q_pos + q_len)
    seg_seq: list          # [n_seg] micro-batch sequence index
    seg_chunk: list        # [n_seg] zigzag chunk id, -1 for locals
    src_row: list          # [n_rows] packed row -> rank-natural source row
    n_dist_seg: int
    dist_rows: int


@dataclass
class MicroBatchPack:
    ranks: list                  # RankPack per CP rank
    pad_rows: int                # P (R22)
    natural_rows: int            # rows of the natural distributed-K/V buffer
    nat_base: dict               # seq -> first natural-dist row
    chunks: list                 # per (seq, c): dict(seq, c, owner, gathered_row, natural_row, len)


def pack_microbatch(lens, assign, N: int) -> MicroBatchPack:
    K = len(lens)
    order = sorted(range(K), key=lambda k: (lens[k], k))
    dist = [k for k in order if assign[k] == -1]
    nat_base, acc = {}, 0
    for k in dist:
        nat_base[k] = acc
        acc += int(lens[k])
    ranks = []
    for j in range(N):
        q_len, q_pos, k_start, k_len, sseq, schunk = [], [], [], [], [], []
        for k in dist:
            for c in (j, 2 * N - 1 - j):
                a, b = chunk_bounds(int(lens[k]), c, N)
                q_len.append(b - a)
                q_pos.append(a)
                k_len.append(b)
                k_start.append(nat_base[k])
                sseq.append(k)
                schunk.append(c)
        n_dist_seg = len(q_len)
        dist_rows = sum(q_len)
        row = dist_rows
        for k in order:
            if assign[k] == j:
                S = int(lens[k])
                q_len.append(S)
                q_pos.append(0)
                k_len.append(S)
                k_start.append(row)
                sseq.append(k)
                schunk.append(-1)
                row += S
        cu = [0]
        for x in q_len:
            cu.append(cu[-1] + x)
        # rank-natural source rows: input-index order, positions ascending
        src_base, s = {}, 0
        for k in range(K):
            if assign[k] == j:
                src_base[(k, -1)] = s
                s += int(lens[k])
            elif assign[k] == -1:
                for c in sorted((j, 2 * N - 1 - j)):
                    a, b = chunk_bounds(int(lens[k]), c, N)
                    src_base[(k, c)] = s
                    s += b - a
        src_row = []
        for i in range(len(q_len)):
            base = src_base[(sseq[i], schunk[i])]
            src_row.extend(range(base, base + q_len[i]))
        ranks.append(RankPack(cu, q_pos, k_start, k_len, sseq, schunk, src_row,
                              n_dist_seg, dist_rows))
    P = max(r.dist_rows for r in ranks) if ranks else 0
    chunks = []
    for k in dist:
        for c in range(2 * N):
            o = chunk_owner(c, N)
            r = ranks[o]
            off = next(r.cu_seqlens_q[i] for i in range(r.n_dist_seg)
                       if r.seg_seq[i] == k and r.seg_chunk[i] == c)
            a, b = chunk_bounds(int(lens[k]), c, N)
            chunks.append(dict(seq=k, c=c, owner=o, gathered_row=o * P + off,
                               natural_row=nat_base[k] + a, len=b - a))
    return MicroBatchPack(ranks, P, acc, nat_base, chunks)
