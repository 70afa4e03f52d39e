"""CP-rank runtime for one DACP micro-batch: buffers, device tables and the launch order of rows
a5-a9 (SURVEY.md §3 stacks 2-3), all through the C-ABI (`skrull.py`).

Forward (Eq. 2, P:156 executed literally):
  main : pack Q,K,V (a5)                                          -> ev_packed
  side : wait ev_packed; all-gather K,V distributed prefix (a6);
         reorder rank-major -> natural distributed order           -> ev_kv
  main : attention fwd over LOCAL segments (overlaps the exchange)
  main : wait ev_kv; attention fwd over DISTRIBUTED chunks
Backward (mirror, reading R24):
  main : pack dO; attention bwd over DISTRIBUTED chunks (fp32 dK/dV partials, natural order) -> ev_dkv
  side : wait ev_dkv; permute natural -> rank-major (a9); reduce-scatter; cast into the packed
         dK/dV distributed prefix                                                          -> ev_rs
  main : attention bwd over LOCAL segments (overlaps the exchange); wait ev_rs
With N = 1 (or no distributed sequence) no collective is issued (T_comm(0) = 0, R26).

Each phase is a method so a test can drive N ranks on one GPU with a loopback exchange
(`loopback_step`); `forward` / `backward` are the production composition over a `Comm`.
"""
from __future__ import annotations

import numpy as np
import torch

from . import skrull as sk


class BufferPool:
    """Working buffers shared by the micro-batches of one rank, which run one after another (the
    Eq. 8 sum over micro-batches): every named buffer is ONE flat allocation sized to the
    largest request, and each RankStep takes views of it. Two phases: RankSteps are built with
    `reserve` (meta-tensor placeholders), then `materialize()` allocates and `RankStep.rebind(pool.get)`
    hands out the views. Keeps a rank's memory at one micro-batch's working set (C5 at 256 sequences
    per GPU needs 57 micro-batches)."""

    def __init__(self, device="cuda"):
        self.dev, self.need, self.bufs = device, {}, None

    def reserve(self, name, shape, dtype):
        n = 1
        for x in shape:
            n *= int(x)
        self.need[name] = (max(self.need.get(name, (0, dtype))[0], n), dtype)
        return torch.empty(shape, dtype=dtype, device="meta")

    def materialize(self):
        # zero-filled: rows past a micro-batch's own rows are read by attention tiles (and multiplied
        # by exact zeros), so they must hold finite values -- zeros here, finite data of a larger
        # micro-batch later
        self.bufs = {k: torch.zeros(n, dtype=dt, device=self.dev) for k, (n, dt) in self.need.items()}

    def get(self, name, shape, dtype):
        n = 1
        for x in shape:
            n *= int(x)
        return self.bufs[name][:n].view(*shape)


def _alloc_new(device):
    # zero-filled for the same reason as BufferPool.materialize: padding rows [rows, max(rows, P))
    # enter the attention tiles and must be finite (0 x NaN would poison dK / dQ / O)
    return lambda name, shape, dtype: torch.zeros(*shape, device=device, dtype=dtype)


class RankStep:
    def __init__(self, shape, mb_lens, assign, cp: int, rank: int, device="cuda", alloc=None, band_rows=None,
                 ring=False):
        """alloc(name, shape, dtype) -> tensor: where the working buffers come from (default: fresh
        allocations; BufferPool.reserve to share them across micro-batches). band_rows: query-band
        height of the backward work lists (skr_tiles_bwd; None = the library's choice). ring: also build
        the tables and buffers of the ring-CP exchange (row f4, forward_ring / backward_ring)."""
        self.shape, self.cp, self.rank = shape, cp, rank
        self.dev = device
        self._alloc = alloc or _alloc_new(device)
        self._bufspec = []
        hq, hkv, d = shape.hq, shape.hkv, shape.d
        self.dt = torch.bfloat16 if shape.dtype == sk.SKR_BF16 else torch.float32
        pr = sk.skr_pack_rank(mb_lens, assign, cp, rank)
        self.pr = pr
        self.rows = pr["n_rows"]
        self.dist_rows = pr["dist_rows"]
        self.P = pr["pad_rows_P"]
        self.nat_rows = pr["natural_rows"]
        self.n_chunks = pr["n_chunks"]
        nd, ns = pr["n_dist_seg"], pr["n_seg"]
        cu, qp, ks, kl = pr["cu_seqlens_q"], pr["q_pos"], pr["k_start"], pr["k_len"]
        self.has_dist = self.nat_rows > 0
        self.events = None          # list -> (kind, start, end) CUDA events around attention calls;
        #                             kind in fwd_local / fwd_dist / bwd_dist / bwd_local
        self.src_row = torch.as_tensor(pr["src_row"]).to(device)
        # segment classes: distributed chunks [0, nd), locals [nd, ns)
        self.dist_f = sk.make_segs(shape, cu[:nd + 1], qp[:nd], ks[:nd], kl[:nd], "fwd", device)
        self.dist_b = sk.make_segs(shape, cu[:nd + 1], qp[:nd], ks[:nd], kl[:nd], "bwd", device, band_rows)
        self.loc_f = sk.make_segs(shape, cu[nd:], qp[nd:], ks[nd:], kl[nd:], "fwd", device)
        self.loc_b = sk.make_segs(shape, cu[nd:], qp[nd:], ks[nd:], kl[nd:], "bwd", device, band_rows)
        if self.has_dist:
            table = sk.skr_pack_chunks(mb_lens, assign, cp)
            self.chunks = torch.as_tensor(table.reshape(-1)).to(device)
            # row f3 step two: natural row -> owner * P + prefix row (skr_attn_bwd_peer)
            self.owner_rows = torch.as_tensor(sk.skr_pack_owner_rows(table, self.nat_rows)).to(device)
        # packed buffers (>= P rows so the all-gather send prefix is always in bounds)
        R = max(self.rows, self.P, 1)
        f32, dt = torch.float32, self.dt
        for name in ("q", "o", "do", "dq"):
            self._buf(name, (R, hq, d), dt)
        for name in ("k", "v", "dk", "dv"):
            self._buf(name, (R, hkv, d), dt)
        self._buf("lse", (hq, R), f32)
        self._buf("ws", (sk.skr_attn_bwd_ws_bytes(shape, R) // 4 + 64,), f32)
        if self.has_dist:
            N, P, nat = cp, self.P, max(self.nat_rows, 1)
            for name in ("k_gath", "v_gath"):
                self._buf(name, (N * P, hkv, d), dt)
            for name in ("k_nat", "v_nat"):
                self._buf(name, (nat, hkv, d), dt)
            for name in ("dk_nat", "dv_nat"):
                self._buf(name, (nat, hkv, d), f32)
            for name in ("dk_rm", "dv_rm"):
                self._buf(name, (N * P, hkv, d), f32)
            for name in ("dk_red", "dv_red"):
                self._buf(name, (P, hkv, d), f32)
            # row f3 step two: this rank's fp32 accumulators of the rows it OWNS (its distributed
            # prefix); every rank's backward red-adds its partials into them over peer memory
            for name in ("dk_acc", "dv_acc"):
                self._buf(name, (max(P, 1), hkv, d), f32)
        self.ring = bool(ring) and self.has_dist
        if self.ring:
            # row f4, ring CP: per hop r and key-chunk class c the segment tables of this rank's query
            # chunks against the visiting prefix (skr_ring_segs), double-buffered visiting K/V and
            # travelling fp32 dK/dV accumulators, the partial O / LSE and the fp32 running O, dQ
            P = max(self.P, 1)
            self.ring_f, self.ring_b = [], []
            for r in range(cp):
                fr, br = [], []
                for c in (0, 1):
                    t = sk.skr_ring_segs(mb_lens, assign, cp, rank, r, c)
                    fr.append(sk.make_segs(shape, t["cu_seqlens_q"], t["q_pos"], t["k_start"], t["k_len"], "fwd",
                                           device))
                    br.append(sk.make_segs(shape, t["cu_seqlens_q"], t["q_pos"], t["k_start"], t["k_len"], "bwd",
                                           device, band_rows))
                self.ring_f.append(fr)
                self.ring_b.append(br)
            for name in ("ring_k0", "ring_k1", "ring_v0", "ring_v1"):
                self._buf(name, (P, hkv, d), dt)
            for name in ("ring_dk0", "ring_dk1", "ring_dv0", "ring_dv1"):
                self._buf(name, (P, hkv, d), f32)
            self._buf("ring_o", (R, hq, d), dt)
            self._buf("ring_lse", (hq, R), f32)
            self._buf("ring_oacc", (R, hq, d), f32)
            self._buf("ring_dq", (R, hq, d), f32)

    def cp_step(self, q_src, k_src, v_src, do_src, timing=None):
        """The skr_cp_step of this micro-batch (row a5-a9 composite C-ABI call) for these inputs.
        timing: optional 8 torch.cuda.Events (already created) the library records around its
        attention calls (skr_cp_step.timing_events)."""
        if getattr(self, "_plan", None) is None:
            self._plan = sk.AttnPlan(self.shape, self.q.shape[0])
        p = lambda t: t.data_ptr() if t is not None else 0  # noqa: E731
        d = self.has_dist
        return sk.skr_cp_step(
            self.loc_f.struct(), self.loc_b.struct(), self.dist_f.struct(), self.dist_b.struct(),
            p(self.chunks) if d else 0, self.n_chunks if d else 0, self.cp, self.rows, self.dist_rows, self.P,
            self.nat_rows, self.q.shape[0], p(self.src_row),
            p(q_src), p(k_src), p(v_src), p(do_src),
            p(self.q), p(self.k), p(self.v), p(self.o), p(self.do), p(self.dq), p(self.dk), p(self.dv), p(self.lse),
            p(self.k_gath) if d else 0, p(self.v_gath) if d else 0, p(self.k_nat) if d else 0,
            p(self.v_nat) if d else 0, p(self.dk_nat) if d else 0, p(self.dv_nat) if d else 0,
            p(self.dk_rm) if d else 0, p(self.dv_rm) if d else 0, p(self.dk_red) if d else 0,
            p(self.dv_red) if d else 0, p(self.ws), self.ws.numel() * 4, self._timing_ptr(timing))

    def _timing_ptr(self, timing):
        if timing is None:
            self._timing_arr = None
            return 0
        import ctypes
        arr = (ctypes.c_void_p * 8)(*[e.cuda_event for e in timing])
        self._timing_arr = arr          # alive for the duration of the call
        return ctypes.addressof(arr)

    def _buf(self, name, shape, dtype):
        self._bufspec.append((name, shape, dtype))
        setattr(self, name, self._alloc(name, shape, dtype))

    def rebind(self, alloc):
        """Re-fetch every working buffer from `alloc` (after BufferPool.materialize)."""
        for name, shape, dtype in self._bufspec:
            setattr(self, name, alloc(name, shape, dtype))

    def launches_per_step(self, exchange="nccl") -> int:
        """Kernels of this library launched by one forward + backward of this micro-batch."""
        n = 0
        if self.rows:
            n += 4                                            # pack Q, K, V, dO
        loc_rows = self.loc_b.row_end - self.loc_b.row_begin
        # local bwd: + the band accumulator zero / cast launches (kv_accumulate = 0)
        n += (self.loc_f.n_tiles > 0) + 3 * (self.loc_b.n_tiles > 0) + 2 * (loc_rows > 0)
        if self.has_dist:
            dist_rows = self.dist_b.row_end - self.dist_b.row_begin
            n += (self.dist_f.n_tiles > 0) + (self.dist_b.n_tiles > 0) + 2 * (dist_rows > 0)
            if exchange == "ring" and self.ring:
                # replaces the all-gather path's distributed launches: per hop and key-chunk class a
                # forward + merge, a D-preprocess + backward (accumulate mode: no dQ convert, no band
                # zero / cast); then the casts of O, dQ, dK, dV
                n -= (self.dist_f.n_tiles > 0) + (self.dist_b.n_tiles > 0) + 2 * (dist_rows > 0)
                for r in range(self.cp):
                    for c in (0, 1):
                        n += (self.ring_f[r][c].n_tiles > 0) + 2 * (dist_rows > 0) + (self.ring_b[r][c].n_tiles > 0)
                n += 4 * (dist_rows > 0 and self.dt != torch.float32)
                return n
            if exchange == "peer":
                # step two: gather K, V; cast dK, dV (the reduction is inside the bwd kernel); 3 signal + wait
                n += 2 + 2 * (self.dist_rows > 0) + 3 * 2
            elif exchange == "peer1":
                n += 2 + 2 + 3 * 2                            # gather K, V; reduce dK, dV; 3 signal + wait
            else:
                n += 2 + 2 + 2 * (self.dist_rows > 0)         # reorder K, V; scatter dK, dV; cast dK, dV
        return n

    # ------------------------------------------------------------------ phases
    def pack_qkv(self, q_src, k_src, v_src, stream=None):
        if self.rows:
            sk.skr_pack_rows(q_src, self.src_row, self.q[:self.rows], stream)
            sk.skr_pack_rows(k_src, self.src_row, self.k[:self.rows], stream)
            sk.skr_pack_rows(v_src, self.src_row, self.v[:self.rows], stream)

    def pack_do(self, do_src, stream=None):
        if self.rows:
            sk.skr_pack_rows(do_src, self.src_row, self.do[:self.rows], stream)

    def kv_send(self):
        return self.k[:self.P], self.v[:self.P]

    def kv_reorder(self, stream=None):
        sk.skr_gather_chunks(self.k_gath, self.chunks, self.n_chunks, self.k_nat, stream)
        sk.skr_gather_chunks(self.v_gath, self.chunks, self.n_chunks, self.v_nat, stream)

    def _timed(self, kind, fn, stream):
        if self.events is None:
            return fn()
        s = stream if stream is not None else torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        self.events.append((kind, e0, e1))

    def fwd_local(self, stream=None):
        self._timed("fwd_local", lambda: sk.skr_attn_fwd(self.shape, self.loc_f, self.q, self.k, self.v, self.o, self.lse,
                                                   stream), stream)

    def fwd_dist(self, stream=None):
        self._timed("fwd_dist", lambda: sk.skr_attn_fwd(self.shape, self.dist_f, self.q, self.k_nat, self.v_nat, self.o,
                                                   self.lse, stream), stream)

    def bwd_dist(self, stream=None):
        self.dk_nat.zero_()
        self.dv_nat.zero_()
        self._timed("bwd_dist", lambda: sk.skr_attn_bwd(self.shape, self.dist_b, self.q, self.k_nat, self.v_nat, self.o,
                                                   self.do, self.lse, self.dq, self.dk_nat, self.dv_nat, 1, self.ws,
                                                   stream), stream)

    def grad_scatter(self, stream=None):
        sk.skr_scatter_chunks(self.dk_nat, self.chunks, self.n_chunks, self.P, self.cp, self.dk_rm, stream)
        sk.skr_scatter_chunks(self.dv_nat, self.chunks, self.n_chunks, self.P, self.cp, self.dv_rm, stream)

    def grad_cast(self, stream=None):
        n = self.dist_rows
        if n:
            if self.dt == torch.float32:
                self.dk[:n].copy_(self.dk_red[:n])
                self.dv[:n].copy_(self.dv_red[:n])
            else:
                sk.skr_cast_f32_bf16(self.dk_red[:n], self.dk[:n], stream)
                sk.skr_cast_f32_bf16(self.dv_red[:n], self.dv[:n], stream)

    def bwd_local(self, stream=None):
        self._timed("bwd_local", lambda: sk.skr_attn_bwd(self.shape, self.loc_b, self.q, self.k, self.v, self.o, self.do,
                                                   self.lse, self.dq, self.dk, self.dv, 0, self.ws, stream), stream)

    # ------------------------------------------------------------------ production composition
    # One C-ABI call per direction (skr_cp_attn_fwd / _bwd, csrc/cuda/cp_step.cu). The per-phase
    # composition below runs the same kernels call by call; it is used when the attention calls are
    # timed individually (self.events) and by the one-GPU loopback tests.
    def forward(self, q_src, k_src, v_src, comm=None, side=None, timing=None):
        """timing: optional list of 8 created torch.cuda.Events (only [0:4] are recorded here)."""
        if self.events is None:
            self._fwd_inputs = (q_src, k_src, v_src)
            sk.skr_cp_attn_fwd(comm, self._plan_or_new(), self.cp_step(q_src, k_src, v_src, None, timing),
                               torch.cuda.current_stream(), side or torch.cuda.current_stream())
            return
        self.forward_phases(q_src, k_src, v_src, comm, side)

    def backward(self, do_src, comm=None, side=None, timing=None):
        """timing: optional list of 8 created torch.cuda.Events (only [4:8] are recorded here)."""
        if self.events is None:
            q_src, k_src, v_src = getattr(self, "_fwd_inputs", (None, None, None))
            sk.skr_cp_attn_bwd(comm, self._plan_or_new(), self.cp_step(q_src, k_src, v_src, do_src, timing),
                               torch.cuda.current_stream(), side or torch.cuda.current_stream())
            return
        self.backward_phases(do_src, comm, side)

    def _plan_or_new(self):
        if getattr(self, "_plan", None) is None:
            self._plan = sk.AttnPlan(self.shape, self.q.shape[0])
        return self._plan

    def forward_phases(self, q_src, k_src, v_src, comm=None, side=None):
        main = torch.cuda.current_stream()
        self.pack_qkv(q_src, k_src, v_src)
        if self.has_dist:
            ev_packed = torch.cuda.Event()
            ev_packed.record(main)
            side.wait_event(ev_packed)
            with torch.cuda.stream(side):
                ks, vs = self.kv_send()
                comm.all_gather(ks, self.k_gath, side)
                comm.all_gather(vs, self.v_gath, side)
                self.kv_reorder(side)
                ev_kv = torch.cuda.Event()
                ev_kv.record(side)
        self.fwd_local()
        if self.has_dist:
            main.wait_event(ev_kv)
            self.fwd_dist()

    def backward_phases(self, do_src, comm=None, side=None):
        main = torch.cuda.current_stream()
        self.pack_do(do_src)
        if self.has_dist:
            self.bwd_dist()
            ev_dkv = torch.cuda.Event()
            ev_dkv.record(main)
            side.wait_event(ev_dkv)
            with torch.cuda.stream(side):
                self.grad_scatter(side)
                comm.reduce_scatter_f32(self.dk_rm, self.dk_red, side)
                comm.reduce_scatter_f32(self.dv_rm, self.dv_red, side)
                self.grad_cast(side)
                ev_rs = torch.cuda.Event()
                ev_rs.record(side)
        self.bwd_local()
        if self.has_dist:
            main.wait_event(ev_rs)


    # ------------------------------------------------------------------ row f4: ring CP
    def ring_bufs(self, r):
        """Visiting K / V buffers of hop r >= 1 (double-buffered; hop 0 visits the own prefix)."""
        i = (r - 1) % 2
        return getattr(self, f"ring_k{i}"), getattr(self, f"ring_v{i}")

    def ring_acc(self, r):
        """Travelling fp32 dK / dV accumulators of hop r (double-buffered)."""
        i = r % 2
        return getattr(self, f"ring_dk{i}"), getattr(self, f"ring_dv{i}")

    def ring_fwd_hop(self, r, vk, vv, stream=None):
        """Hop r of the ring forward: this rank's query chunks against the visiting prefix (vk, vv),
        one partial attention per key chunk of the pair, each merged into the running (O, LSE)."""
        n = self.dist_rows
        for c in (0, 1):
            self._timed("fwd_dist", lambda c=c: sk.skr_attn_fwd(self.shape, self.ring_f[r][c], self.q, vk, vv,
                                                              self.ring_o, self.ring_lse, stream), stream)
            sk.skr_attn_merge(self.shape, self.ring_o, self.ring_lse, self.ring_oacc, self.lse, 0, n,
                              r == 0 and c == 0, stream)

    def ring_fwd_finish(self, stream=None):
        n = self.dist_rows
        if self.dt == torch.float32:
            s = stream if stream is not None else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                self.o[:n].copy_(self.ring_oacc[:n])
        else:
            sk.skr_cast_f32_bf16(self.ring_oacc[:n], self.o[:n], stream)

    def ring_bwd_start(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.ring_dq[:self.dist_rows].zero_()
            for t in self.ring_acc(0):
                t.zero_()

    def ring_bwd_hop(self, r, vk, vv, stream=None):
        """Hop r of the ring backward: dQ of this rank's query chunks accumulates in fp32, the visiting
        chunks' dK / dV are added into the travelling accumulators (final O / LSE of the forward)."""
        ak, av = self.ring_acc(r)
        for c in (0, 1):
            self._timed("bwd_dist", lambda c=c: sk.skr_attn_bwd_acc(
                self.shape, self.ring_b[r][c], self.q, vk, vv, self.o, self.do, self.lse, self.ring_dq, ak, av,
                self.ws, stream), stream)

    def ring_bwd_finish(self, stream=None):
        """After N accumulator hops this rank holds its own chunks' summed dK / dV."""
        n = self.dist_rows
        ak, av = self.ring_acc(self.cp)
        if self.dt == torch.float32:
            s = stream if stream is not None else torch.cuda.current_stream()
            with torch.cuda.stream(s):
                self.dq[:n].copy_(self.ring_dq[:n])
                self.dk[:n].copy_(ak[:n])
                self.dv[:n].copy_(av[:n])
        else:
            sk.skr_cast_f32_bf16(self.ring_dq[:n], self.dq[:n], stream)
            sk.skr_cast_f32_bf16(ak[:n], self.dk[:n], stream)
            sk.skr_cast_f32_bf16(av[:n], self.dv[:n], stream)

    def forward_ring(self, q_src, k_src, v_src, comm, side):
        """Eq. 2 with the ring exchange: main packs and runs the LOCAL tiles while the side stream
        moves the own prefix one hop; then per hop r main computes against the visiting prefix while
        the side stream moves it on (double-buffered; a receive buffer is reused only after the hop
        that read it)."""
        main = torch.cuda.current_stream()
        self.pack_qkv(q_src, k_src, v_src)
        if not self.has_dist:
            self.fwd_local()
            return
        N, P = self.cp, self.P
        cur = (self.k[:P], self.v[:P])
        ev_cur = torch.cuda.Event()
        ev_cur.record(main)
        done = [None] * N
        recv = None
        for r in range(N):
            if r + 1 < N:
                nxt = self.ring_bufs(r + 1)
                side.wait_event(ev_cur)
                if r >= 1:
                    side.wait_event(done[r - 1])     # nxt was the visiting buffer of hop r - 1
                with torch.cuda.stream(side):
                    comm.ring_shift([cur[0], cur[1]], [nxt[0][:P], nxt[1][:P]], side)
                    recv = torch.cuda.Event()
                    recv.record(side)
            if r == 0:
                self.fwd_local()
            self.ring_fwd_hop(r, cur[0], cur[1])
            done[r] = torch.cuda.Event()
            done[r].record(main)
            if r + 1 < N:
                main.wait_event(recv)
                cur, ev_cur = (nxt[0][:P], nxt[1][:P]), recv
        self.ring_fwd_finish()

    def backward_ring(self, do_src, comm, side):
        """Mirror: per hop r main computes dQ (fp32, accumulated) and the visiting chunks' dK / dV
        (into the travelling accumulators); the side stream moves the visiting K / V on during the
        hop and the accumulators after it; after N accumulator hops they are home. LOCAL tiles run on
        main after the first hop's kernels."""
        main = torch.cuda.current_stream()
        self.pack_do(do_src)
        if not self.has_dist:
            self.bwd_local()
            return
        N, P = self.cp, self.P
        self.ring_bwd_start()
        cur = (self.k[:P], self.v[:P])
        ev_cur = torch.cuda.Event()
        ev_cur.record(main)
        done = [None] * N
        for r in range(N):
            kv_recv = None
            if r + 1 < N:
                nxt = self.ring_bufs(r + 1)
                side.wait_event(ev_cur)
                if r >= 1:
                    side.wait_event(done[r - 1])
                with torch.cuda.stream(side):
                    comm.ring_shift([cur[0], cur[1]], [nxt[0][:P], nxt[1][:P]], side)
                    kv_recv = torch.cuda.Event()
                    kv_recv.record(side)
            self.ring_bwd_hop(r, cur[0], cur[1])
            done[r] = torch.cuda.Event()
            done[r].record(main)
            # the accumulators carry this hop's contribution on to the next rank (N hops: home)
            side.wait_event(done[r])
            with torch.cuda.stream(side):
                (ak, av), (bk, bv) = self.ring_acc(r), self.ring_acc(r + 1)
                comm.ring_shift([ak[:P], av[:P]], [bk[:P], bv[:P]], side)
                acc_recv = torch.cuda.Event()
                acc_recv.record(side)
            if r == 0:
                self.bwd_local()
            main.wait_event(acc_recv)
            if kv_recv is not None:
                main.wait_event(kv_recv)
                cur, ev_cur = (nxt[0][:P], nxt[1][:P]), kv_recv
        self.ring_bwd_finish()

    # ------------------------------------------------------------------ row f3: peer-memory exchange
    def connect_peer(self, peer):
        """Collective over the CP group: map the peers' packed K/V, natural fp32 dK/dV partials (step
        one) and owned fp32 dK/dV accumulators (step two)."""
        self.peer = peer
        if self.has_dist:
            self.peer_k, self.peer_v, self.peer_dk, self.peer_dv, self.peer_dk_acc, self.peer_dv_acc = peer.exchange(
                [self.k, self.v, self.dk_nat, self.dv_nat, self.dk_acc, self.dv_acc])

    def peer_gather(self, stream=None):
        sk.skr_peer_gather_chunks(self.peer_k, self.chunks, self.n_chunks, self.P, self.k_nat, stream)
        sk.skr_peer_gather_chunks(self.peer_v, self.chunks, self.n_chunks, self.P, self.v_nat, stream)

    def peer_reduce(self, stream=None):
        re = self.shape.hkv * self.shape.d
        sk.skr_peer_reduce_chunks(self.peer_dk, self.cp, self.rank, self.chunks, self.n_chunks, re, self.P,
                                  self.dk, stream)
        sk.skr_peer_reduce_chunks(self.peer_dv, self.cp, self.rank, self.chunks, self.n_chunks, re, self.P,
                                  self.dv, stream)

    def bwd_dist_fused(self, stream=None):
        """Row f3 step two: the distributed chunks' backward red-adds its dK/dV partials straight into
        the OWNERS' fp32 accumulators (peer memory) from the kernel epilogue."""
        self._timed("bwd_dist", lambda: sk.skr_attn_bwd_peer(
            self.shape, self.dist_b, self.q, self.k_nat, self.v_nat, self.o, self.do, self.lse, self.dq,
            self.peer_dk_acc, self.peer_dv_acc, self.owner_rows, self.P, self.ws, stream), stream)

    def acc_zero(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.dk_acc.zero_()
            self.dv_acc.zero_()

    def acc_cast(self, stream=None):
        """Owner side: the summed fp32 rows of this rank's distributed prefix -> packed dK/dV."""
        n = self.dist_rows
        if n:
            if self.dt == torch.float32:
                s = stream if stream is not None else torch.cuda.current_stream()
                with torch.cuda.stream(s):
                    self.dk[:n].copy_(self.dk_acc[:n])
                    self.dv[:n].copy_(self.dv_acc[:n])
            else:
                sk.skr_cast_f32_bf16(self.dk_acc[:n], self.dk[:n], stream)
                sk.skr_cast_f32_bf16(self.dv_acc[:n], self.dv[:n], stream)

    def backward_peer_fused(self, do_src, side):
        """Mirror of Eq. 2 (R24) with the a9 exchange fused into the a8 kernel (row f3 step two):
        main: pack dO; zero the owned accumulators; epoch 'zeroed' (all ranks); distributed backward
        (red-adds into the owners' accumulators over NVLink); epoch 'added'; side: wait for every
        rank's 'added', cast the owned rows into the packed bf16 dK/dV prefix, while main runs the
        local tiles. A rank zeroes its accumulators for the next micro-batch only after its cast
        (main waits for the side stream), and the others add into them only after the next
        'zeroed' epoch, so no extra 'consumed' epoch is needed."""
        main = torch.cuda.current_stream()
        self.pack_do(do_src)
        if self.has_dist:
            self.acc_zero(main)
            e = self.peer.signal(main)
            self.peer.wait(e, main)
            self.bwd_dist_fused()
            e2 = self.peer.signal(main)
            with torch.cuda.stream(side):
                self.peer.wait(e2, side)
                self.acc_cast(side)
                ev_rs = torch.cuda.Event()
                ev_rs.record(side)
        self.bwd_local()
        if self.has_dist:
            main.wait_event(ev_rs)

    def forward_peer(self, q_src, k_src, v_src, side):
        """Eq. 2 with the a6 exchange as one peer-gather pass: pack; signal 'packed K/V ready'; on the
        side stream wait for every peer, then copy each distributed chunk from its owner's packed
        buffer into the natural buffer, while the main stream runs the local tiles."""
        main = torch.cuda.current_stream()
        self.pack_qkv(q_src, k_src, v_src)
        if self.has_dist:
            e = self.peer.signal(main)
            with torch.cuda.stream(side):
                self.peer.wait(e, side)
                self.peer_gather(side)
                ev_kv = torch.cuda.Event()
                ev_kv.record(side)
        self.fwd_local()
        if self.has_dist:
            main.wait_event(ev_kv)
            self.fwd_dist()

    def backward_peer(self, do_src, side):
        """Mirror (R24): distributed tiles first; signal 'partials ready'; on the side stream wait,
        sum every owned chunk over the peers' partials straight into the packed bf16 dK/dV prefix,
        then a second epoch ('partials consumed') before the buffers may be reused."""
        main = torch.cuda.current_stream()
        self.pack_do(do_src)
        if self.has_dist:
            self.bwd_dist()
            e = self.peer.signal(main)
            with torch.cuda.stream(side):
                self.peer.wait(e, side)
                self.peer_reduce(side)
                e2 = self.peer.signal(side)
                self.peer.wait(e2, side)
                ev_rs = torch.cuda.Event()
                ev_rs.record(side)
        self.bwd_local()
        if self.has_dist:
            main.wait_event(ev_rs)


def loopback_peer_step(ranks, q_srcs, k_srcs, v_srcs, do_srcs):
    """Row f3 on ONE GPU in one process: the peer-gather / peer-reduce kernels with the other
    emulated ranks' buffers as the 'peer' addresses (no flags needed: the ranks run in order)."""
    N = len(ranks)
    for r, x in enumerate(ranks):
        x.pack_qkv(q_srcs[r], k_srcs[r], v_srcs[r])
        x.pack_do(do_srcs[r])
    if ranks[0].has_dist:
        addr = lambda name: torch.tensor([getattr(y, name).data_ptr() for y in ranks], dtype=torch.int64,  # noqa: E731
                                         device=ranks[0].dev)
        for x in ranks:
            x.peer_k, x.peer_v, x.peer_dk, x.peer_dv = addr("k"), addr("v"), addr("dk_nat"), addr("dv_nat")
            x.peer_gather()
    for x in ranks:
        x.fwd_local()
        if x.has_dist:
            x.fwd_dist()
    if ranks[0].has_dist:
        for x in ranks:
            x.bwd_dist()
        for x in ranks:
            x.peer_reduce()
    for x in ranks:
        x.bwd_local()
    del N
    return ranks


def loopback_peer_fused_step(ranks, q_srcs, k_srcs, v_srcs, do_srcs):
    """Row f3 step two on ONE GPU in one process: the peer gather for the forward, and the
    distributed backward red-adding into the other emulated ranks' owned accumulators (their
    addresses as the 'peer' table); the ranks run in order, so no flags are needed."""
    for r, x in enumerate(ranks):
        x.pack_qkv(q_srcs[r], k_srcs[r], v_srcs[r])
        x.pack_do(do_srcs[r])
    if ranks[0].has_dist:
        addr = lambda name: torch.tensor([getattr(y, name).data_ptr() for y in ranks], dtype=torch.int64,  # noqa: E731
                                         device=ranks[0].dev)
        for x in ranks:
            x.peer_k, x.peer_v = addr("k"), addr("v")
            x.peer_dk_acc, x.peer_dv_acc = addr("dk_acc"), addr("dv_acc")
            x.peer_gather()
    for x in ranks:
        x.fwd_local()
        if x.has_dist:
            x.fwd_dist()
    if ranks[0].has_dist:
        for x in ranks:
            x.acc_zero()
        for x in ranks:
            x.bwd_dist_fused()
        for x in ranks:
            x.acc_cast()
    for x in ranks:
        x.bwd_local()
    return ranks


def loopback_ring_step(ranks, q_srcs, k_srcs, v_srcs, do_srcs):
    """Row f4 ring CP on ONE GPU in one process: the N emulated ranks run each hop in lockstep, the
    ring hops (point-to-point sends) replaced by device copies. Same kernels and tables as the
    NCCL ring (RankStep.forward_ring / backward_ring)."""
    N = len(ranks)
    for r, x in enumerate(ranks):
        x.pack_qkv(q_srcs[r], k_srcs[r], v_srcs[r])
        x.pack_do(do_srcs[r])
    for x in ranks:
        x.fwd_local()
    if ranks[0].has_dist:
        P = ranks[0].P
        vis = [(x.k[:P], x.v[:P]) for x in ranks]
        for r in range(N):
            for x, (vk, vv) in zip(ranks, vis):
                x.ring_fwd_hop(r, vk, vv)
            if r + 1 < N:   # hop: rank j receives rank j - 1's visiting prefix
                nxt = []
                for j, x in enumerate(ranks):
                    bk, bv = x.ring_bufs(r + 1)
                    bk[:P].copy_(vis[(j - 1) % N][0])
                    bv[:P].copy_(vis[(j - 1) % N][1])
                    nxt.append((bk[:P], bv[:P]))
                vis = nxt
        for x in ranks:
            x.ring_fwd_finish()
        for x in ranks:
            x.ring_bwd_start()
        vis = [(x.k[:P], x.v[:P]) for x in ranks]
        for r in range(N):
            for x, (vk, vv) in zip(ranks, vis):
                x.ring_bwd_hop(r, vk, vv)
            for j, x in enumerate(ranks):   # accumulator hop (also after the last: home)
                bk, bv = x.ring_acc(r + 1)
                ak, av = ranks[(j - 1) % N].ring_acc(r)
                bk[:P].copy_(ak[:P])
                bv[:P].copy_(av[:P])
            if r + 1 < N:
                nxt = []
                for j, x in enumerate(ranks):
                    bk, bv = x.ring_bufs(r + 1)
                    bk[:P].copy_(vis[(j - 1) % N][0])
                    bv[:P].copy_(vis[(j - 1) % N][1])
                    nxt.append((bk[:P], bv[:P]))
                vis = nxt
        for x in ranks:
            x.ring_bwd_finish()
    for x in ranks:
        x.bwd_local()
    return ranks


def loopback_step(ranks, q_srcs, k_srcs, v_srcs, do_srcs):
    """Debug aid: run N RankSteps of one micro-batch on ONE GPU, the all-gather and
    reduce-scatter replaced by device copies. Same kernels and tables as production."""
    N = len(ranks)
    for r, x in enumerate(ranks):
        x.pack_qkv(q_srcs[r], k_srcs[r], v_srcs[r])
        x.pack_do(do_srcs[r])
    if ranks[0].has_dist:
        P = ranks[0].P
        for x in ranks:
            for j, y in enumerate(ranks):
                ks, vs = y.kv_send()
                x.k_gath[j * P:(j + 1) * P].copy_(ks)
                x.v_gath[j * P:(j + 1) * P].copy_(vs)
            x.kv_reorder()
    for x in ranks:
        x.fwd_local()
        if x.has_dist:
            x.fwd_dist()
    if ranks[0].has_dist:
        for x in ranks:
            x.bwd_dist()
            x.grad_scatter()
        P = ranks[0].P
        for j, x in enumerate(ranks):
            x.dk_red.copy_(sum(y.dk_rm[j * P:(j + 1) * P] for y in ranks))
            x.dv_red.copy_(sum(y.dv_rm[j * P:(j + 1) * P] for y in ranks))
            x.grad_cast()
    for x in ranks:
        x.bwd_local()
    del N
    return ranks


def rank_natural_rows(lens, assign, cp, rank):
    """Rows of this rank's rank-natural source buffer as (seq, lo, hi) position ranges, in order
    (input order; a distributed sequence contributes chunk min(j, 2N-1-j) then max)."""
    out = []
    for k, S in enumerate(lens):
        S = int(S)
        if assign[k] == rank:
            out.append((k, 0, S))
        elif assign[k] == -1:
            for c in sorted((rank, 2 * cp - 1 - rank)):
                out.append((k, c * S // (2 * cp), (c + 1) * S // (2 * cp)))
    return out


def gather_rank_natural(per_seq, lens, assign, cp, rank, key):
    """Concatenate per-sequence arrays (numpy [S, H, d]) into this rank's rank-natural buffer."""
    parts = [per_seq[k][key][lo:hi] for k, lo, hi in rank_natural_rows(lens, assign, cp, rank)]
    if not parts:
        return np.zeros((0,) + per_seq[0][key].shape[1:], np.float32)
    return np.concatenate(parts, axis=0)


def grid_coords(rank: int, world: int, dp: int):
    """DP x CP grid: rank -> (dp_rank, cp_rank, cp). CP groups are blocks of
    cp consecutive ranks (one NVSwitch domain), DP ranks stride over them; GDS / LPT bins are per DP
    rank (Alg. 2 line 1) and DACP places inside each CP group (Alg. 1)."""
    if dp < 1 or world % dp:
        raise ValueError(f"world {world} is not a multiple of dp {dp}")
    cp = world // dp
    return rank // cp, rank % cp, cp


def dp_micro_batches(plan, lens, dp_rank: int):
    """Micro-batches of one DP rank from skr_plan's output, in order: list of (seq indices, lens, assign)."""
    lens = np.asarray(lens)
    out = []
    for j in range(int(plan["n_mb_per_dp"][dp_rank])):
        idx = np.nonzero((plan["dp_of_seq"] == dp_rank) & (plan["mb_of_seq"] == j))[0]
        out.append((idx, lens[idx], plan["assign"][idx]))
    return out
