"""Thin ctypes binding of libskrull.so (include/skrull.h): same names, marshalling only.

Host planner calls take Python sequences / numpy arrays and return numpy arrays. Device calls
take torch tensors (device memory) and use the current torch CUDA stream unless `stream` is
given. Every non-OK status raises SkrullError with skr_last_error()'s message. There is no
fallback: if the library is missing this module fails to import.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKR_LIB_PATH: load another in-tree build of the same library (A/B performance experiments)
LIB_PATH = os.environ.get("SKR_LIB_PATH") or os.path.join(_HERE, "libskrull.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2505_19609_b200.build`")

_lib = C.CDLL(LIB_PATH)

SKR_OK, SKR_E_ARG, SKR_E_SCHEDULE, SKR_E_GDS, SKR_E_BUDGET, SKR_E_PROFILE = range(6)
SKR_E_OVERFLOW, SKR_E_CAPACITY, SKR_E_CUDA, SKR_E_NCCL, SKR_E_UNSUPPORTED = range(6, 11)
SKR_BF16, SKR_FP32 = 0, 1

i32, i64, f64, f32 = C.c_int32, C.c_int64, C.c_double, C.c_float
P = C.POINTER
vp = C.c_void_p


class SkrullError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class skr_model(C.Structure):
    _fields_ = [("hidden", i64), ("kv_hidden", i64), ("pack_batch", i64)]


class skr_fit(C.Structure):
    _fields_ = [("slope", f64), ("intercept", f64)]


class skr_cost(C.Structure):
    _fields_ = [("comp", skr_fit), ("comm", skr_fit), ("mem", skr_fit), ("bytes_per_elem", f64),
                ("dist_penalty", f64)]


class skr_cluster(C.Structure):
    _fields_ = [("cp", i32), ("dp", i32), ("bucket_tokens", i64), ("rollback", i32)]


class skr_attn_shape(C.Structure):
    _fields_ = [("hq", i32), ("hkv", i32), ("d", i32), ("dtype", i32), ("scale", f32)]


class skr_segs(C.Structure):
    _fields_ = [("cu_seqlens_q", vp), ("q_pos", vp), ("k_start", vp), ("k_len", vp), ("tiles", vp),
                ("n_seg", i32), ("n_tiles", i32), ("row_begin", i32), ("row_end", i32)]


_SIGS = {}


def _sig(name, res, *args):
    """The library function `name` with its ctypes prototype, declared once per process (the
    per-call RankStep path would otherwise re-declare prototypes on every call)."""
    fn = _SIGS.get(name)
    if fn is None:
        fn = getattr(_lib, name)
        fn.restype = res
        fn.argtypes = list(args)
        _SIGS[name] = fn
    return fn


_lib.skr_last_error.restype = C.c_char_p
_lib.skr_status_string.restype = C.c_char_p
_lib.skr_status_string.argtypes = [i32]


def _check(st):
    if st != SKR_OK:
        msg = _lib.skr_last_error().decode() or _lib.skr_status_string(st).decode()
        raise SkrullError(st, msg)


def _ptr(a, ctype):
    return a.ctypes.data_as(P(ctype))


def _tptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


def skr_abi_version() -> int:
    return _sig("skr_abi_version", i32)()


# ---------------------------------------------------------------------------- diagnostics
def skr_selftest_umma(variant: int, n: int, A, B, Cout, stream=None):
    fn = _sig("skr_selftest_umma", i32, i32, i32, vp, vp, vp, vp)
    _check(fn(variant, n, _tptr(A), _tptr(B), _tptr(Cout), _stream(stream)))


def exported_symbols():
    """Names the header declares that this library exports (used by the ABI test)."""
    out = []
    for name in _declared_names():
        try:
            getattr(_lib, name)
            out.append(name)
        except AttributeError:
            pass
    return out


def _declared_names():
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "skrull.h")
    with open(hdr) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(skr_[a-z0-9_]+)\s*\(", text)))


# ---------------------------------------------------------------------------- a1 cost model
def _model(hidden, kv_hidden, pack_batch=1):
    return skr_model(int(hidden), int(kv_hidden), int(pack_batch))


def skr_flops(S, hidden, kv_hidden, pack_batch=1) -> int:
    out = i64()
    _check(_sig("skr_flops", i32, i64, P(skr_model), P(i64))(int(S), C.byref(_model(hidden, kv_hidden, pack_batch)),
                                                            C.byref(out)))
    return out.value


def skr_volume(S, hidden, kv_hidden, pack_batch=1) -> int:
    out = i64()
    _check(_sig("skr_volume", i32, i64, P(skr_model), P(i64))(int(S), C.byref(_model(hidden, kv_hidden, pack_batch)),
                                                             C.byref(out)))
    return out.value


def skr_t_comp(flops, slope, intercept) -> float:
    return _sig("skr_t_comp", f64, f64, P(skr_fit))(float(flops), C.byref(skr_fit(slope, intercept)))


def skr_t_comm(volume, slope, intercept) -> float:
    return _sig("skr_t_comm", f64, f64, P(skr_fit))(float(volume), C.byref(skr_fit(slope, intercept)))


def skr_fit_linear(x, y, min_x=0.0):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = skr_fit()
    _check(_sig("skr_fit_linear", i32, P(f64), P(f64), i32, f64, P(skr_fit))(
        _ptr(x, f64), _ptr(y, f64), len(x), float(min_x), C.byref(out)))
    return out.slope, out.intercept


def skr_bucket_size(budget, slope, intercept) -> int:
    out = i64()
    _check(_sig("skr_bucket_size", i32, f64, P(skr_fit), P(i64))(float(budget), C.byref(skr_fit(slope, intercept)),
                                                                C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------- a2/a3 schedulers
def _cluster(cp, dp, bucket, rollback=True):
    return skr_cluster(int(cp), int(dp), int(bucket), 1 if rollback else 0)


def skr_dacp(lens, bucket, cp, hidden, kv_hidden, pack_batch=1, rollback=True):
    """-> (assign int32[K], n_rollbacks). Raises SkrullError(SKR_E_SCHEDULE) with .fail_idx."""
    L = np.ascontiguousarray(lens, np.int64)
    A = np.zeros(len(L), np.int32)
    nrb, fidx = i32(), i32()
    st = _sig("skr_dacp", i32, P(i64), i32, P(skr_cluster), P(skr_model), P(i32), P(i32), P(i32))(
        _ptr(L, i64), len(L), C.byref(_cluster(cp, 1, bucket, rollback)),
        C.byref(_model(hidden, kv_hidden, pack_batch)), _ptr(A, i32), C.byref(nrb), C.byref(fidx))
    if st != SKR_OK:
        e = SkrullError(st, _lib.skr_last_error().decode())
        e.fail_idx = fidx.value
        raise e
    return A, nrb.value


def skr_eval_tdacp(lens, assign, bucket, cp, hidden, kv_hidden, comp, comm, pack_batch=1, bytes_per_elem=1.0,
                   dist_penalty=1.0, mem=(1.0, 0.0)):
    L = np.ascontiguousarray(lens, np.int64)
    A = np.ascontiguousarray(assign, np.int32)
    per = np.zeros(cp, np.float64)
    tc, td, t, feas = f64(), f64(), f64(), i32()
    cost = skr_cost(skr_fit(*comp), skr_fit(*comm), skr_fit(*mem), float(bytes_per_elem), float(dist_penalty))
    _check(_sig("skr_eval_tdacp", i32, P(i64), P(i32), i32, P(skr_cluster), P(skr_model), P(skr_cost), P(f64),
                P(f64), P(f64), P(f64), P(i32))(
        _ptr(L, i64), _ptr(A, i32), len(L), C.byref(_cluster(cp, 1, bucket)),
        C.byref(_model(hidden, kv_hidden, pack_batch)), C.byref(cost), _ptr(per, f64), C.byref(tc), C.byref(td),
        C.byref(t), C.byref(feas)))
    return dict(per_rank_time=per, comm_time=tc.value, dist_time=td.value, tdacp=t.value, feasible=bool(feas.value))


def skr_lpt(lens, bins, hidden, kv_hidden, pack_batch=1):
    L = np.ascontiguousarray(lens, np.int64)
    B = np.zeros(len(L), np.int32)
    _check(_sig("skr_lpt", i32, P(i64), i32, i32, P(skr_model), P(i32))(
        _ptr(L, i64), len(L), int(bins), C.byref(_model(hidden, kv_hidden, pack_batch)), _ptr(B, i32)))
    return B


def skr_gds(lens, bucket, cp, dp, dp_rank, hidden, kv_hidden, pack_batch=1, rollback=True):
    L = np.ascontiguousarray(lens, np.int64)
    M = np.zeros(len(L), np.int32)
    n = i32()
    _check(_sig("skr_gds", i32, P(i64), i32, P(skr_cluster), P(skr_model), i32, P(i32), P(i32))(
        _ptr(L, i64), len(L), C.byref(_cluster(cp, dp, bucket, rollback)),
        C.byref(_model(hidden, kv_hidden, pack_batch)), int(dp_rank), _ptr(M, i32), C.byref(n)))
    return M, n.value


def skr_plan(lens, bucket, cp, dp, hidden, kv_hidden, pack_batch=1, rollback=True):
    """-> dict(dp_of_seq, mb_of_seq, assign, n_mb_per_dp, n_rollbacks)."""
    L = np.ascontiguousarray(lens, np.int64)
    K = len(L)
    dpo, mbo, asg = (np.zeros(K, np.int32) for _ in range(3))
    nmb = np.zeros(dp, np.int32)
    nrb = i32()
    _check(_sig("skr_plan", i32, P(i64), i32, P(skr_cluster), P(skr_model), P(i32), P(i32), P(i32), P(i32),
                P(i32))(
        _ptr(L, i64), K, C.byref(_cluster(cp, dp, bucket, rollback)), C.byref(_model(hidden, kv_hidden, pack_batch)),
        _ptr(dpo, i32), _ptr(mbo, i32), _ptr(asg, i32), _ptr(nmb, i32), C.byref(nrb)))
    return dict(dp_of_seq=dpo, mb_of_seq=mbo, assign=asg, n_mb_per_dp=nmb, n_rollbacks=nrb.value)


def skr_round_robin(lens, bucket, cp, rollback=True):
    """Alg. 4 baseline -> (assign int32[K], n_rollbacks)."""
    L = np.ascontiguousarray(lens, np.int64)
    A = np.zeros(len(L), np.int32)
    nrb, fidx = i32(), i32()
    st = _sig("skr_round_robin", i32, P(i64), i32, P(skr_cluster), P(i32), P(i32), P(i32))(
        _ptr(L, i64), len(L), C.byref(_cluster(cp, 1, bucket, rollback)), _ptr(A, i32), C.byref(nrb), C.byref(fidx))
    if st != SKR_OK:
        e = SkrullError(st, _lib.skr_last_error().decode())
        e.fail_idx = fidx.value
        raise e
    return A, nrb.value


def skr_full_shard(lens, bucket, cp):
    """Full-shard baseline -> (mb_of_seq int32[K], n_mb); every sequence is distributed."""
    L = np.ascontiguousarray(lens, np.int64)
    M = np.zeros(len(L), np.int32)
    n = i32()
    _check(_sig("skr_full_shard", i32, P(i64), i32, P(skr_cluster), P(i32), P(i32))(
        _ptr(L, i64), len(L), C.byref(_cluster(cp, 1, bucket)), _ptr(M, i32), C.byref(n)))
    return M, n.value


# ---------------------------------------------------------------------------- a4 packer
def skr_pack_bounds(mb_lens, assign, cp, rank):
    L = np.ascontiguousarray(mb_lens, np.int64)
    A = np.ascontiguousarray(assign, np.int32)
    v = [i32() for _ in range(7)]
    _check(_sig("skr_pack_bounds", i32, P(i64), P(i32), i32, i32, i32, *([P(i32)] * 7))(
        _ptr(L, i64), _ptr(A, i32), len(L), int(cp), int(rank), *[C.byref(x) for x in v]))
    keys = ("n_seg", "n_dist_seg", "n_rows", "dist_rows", "pad_rows_P", "natural_rows", "n_chunks")
    return dict(zip(keys, (x.value for x in v)))


def skr_pack_rank(mb_lens, assign, cp, rank):
    b = skr_pack_bounds(mb_lens, assign, cp, rank)
    L = np.ascontiguousarray(mb_lens, np.int64)
    A = np.ascontiguousarray(assign, np.int32)
    ns, nr = b["n_seg"], b["n_rows"]
    cu = np.zeros(ns + 1, np.int32)
    qp, ks, kl, ss, sc = (np.zeros(ns, np.int32) for _ in range(5))
    src = np.zeros(nr, np.int32)
    _check(_sig("skr_pack_rank", i32, P(i64), P(i32), i32, i32, i32, *([P(i32)] * 7))(
        _ptr(L, i64), _ptr(A, i32), len(L), int(cp), int(rank), _ptr(cu, i32), _ptr(qp, i32), _ptr(ks, i32),
        _ptr(kl, i32), _ptr(ss, i32), _ptr(sc, i32), _ptr(src, i32)))
    b.update(cu_seqlens_q=cu, q_pos=qp, k_start=ks, k_len=kl, seg_seq=ss, seg_chunk=sc, src_row=src)
    return b


def skr_pack_chunks(mb_lens, assign, cp):
    b = skr_pack_bounds(mb_lens, assign, cp, 0)
    L = np.ascontiguousarray(mb_lens, np.int64)
    A = np.ascontiguousarray(assign, np.int32)
    t = np.zeros((b["n_chunks"], 6), np.int32)
    _check(_sig("skr_pack_chunks", i32, P(i64), P(i32), i32, i32, P(i32))(
        _ptr(L, i64), _ptr(A, i32), len(L), int(cp), _ptr(t, i32)))
    return t


def _tiles(fn_name, cu, q_pos, k_len, n_seg, block, band_rows=0):
    cu = np.ascontiguousarray(cu, np.int32)
    qp = np.ascontiguousarray(q_pos, np.int32)
    width = 2 if fn_name == "skr_tiles_fwd" else 4     # {seg, tile} / {seg, key tile, q_lo, q_hi}
    n = i32()
    cap = 0
    for _ in range(2):
        out = np.zeros(width * max(cap, 1), np.int32)
        if fn_name == "skr_tiles_fwd":
            st = _sig(fn_name, i32, P(i32), P(i32), i32, i32, P(i32), i32, P(i32))(
                _ptr(cu, i32), _ptr(qp, i32), int(n_seg), int(block), _ptr(out, i32), cap, C.byref(n))
        else:
            kl = np.ascontiguousarray(k_len, np.int32)
            st = _sig(fn_name, i32, P(i32), P(i32), P(i32), i32, i32, i32, P(i32), i32, P(i32))(
                _ptr(cu, i32), _ptr(qp, i32), _ptr(kl, i32), int(n_seg), int(block), int(band_rows), _ptr(out, i32),
                cap, C.byref(n))
        if st == SKR_OK:
            return out[:width * n.value].reshape(-1, width)
        if st != SKR_E_CAPACITY:
            _check(st)
        cap = n.value
    raise SkrullError(SKR_E_CAPACITY, "tiles")


def skr_tiles_fwd(cu, q_pos, n_seg, block_m):
    return _tiles("skr_tiles_fwd", cu, q_pos, None, n_seg, block_m)


def skr_tiles_bwd(cu, q_pos, k_len, n_seg, block_n, band_rows=0):
    return _tiles("skr_tiles_bwd", cu, q_pos, k_len, n_seg, block_n, band_rows)


# ---------------------------------------------------------------------------- a5-a9 device
def attn_shape(hq, hkv, d, dtype=SKR_BF16, scale=None):
    return skr_attn_shape(int(hq), int(hkv), int(d), int(dtype), float(scale if scale is not None else d ** -0.5))


def skr_attn_block_m(shape) -> int:
    return _sig("skr_attn_block_m", i32, P(skr_attn_shape))(C.byref(shape))


def skr_attn_block_n(shape) -> int:
    return _sig("skr_attn_block_n", i32, P(skr_attn_shape))(C.byref(shape))


def skr_attn_bwd_band_rows(shape) -> int:
    return _sig("skr_attn_bwd_band_rows", i32, P(skr_attn_shape))(C.byref(shape))


def skr_attn_bwd_ws_bytes(shape, n_q_rows) -> int:
    return _sig("skr_attn_bwd_ws_bytes", C.c_size_t, P(skr_attn_shape), i32)(C.byref(shape), int(n_q_rows))


class DeviceSegs:
    """Device copy of one segment class's tables (+ work list); keeps the tensors alive."""

    def __init__(self, cu, q_pos, k_start, k_len, tiles, row_begin=None, row_end=None, device="cuda"):
        import torch
        cu = np.ascontiguousarray(cu, np.int32)
        self.n_seg = len(cu) - 1
        t = lambda x: torch.as_tensor(np.ascontiguousarray(x, np.int32)).to(device)  # noqa: E731
        self.cu, self.q_pos, self.k_start, self.k_len = t(cu), t(q_pos), t(k_start), t(k_len)
        tiles = np.asarray(tiles, np.int32)
        self.tiles = t(tiles.reshape(-1))
        self.n_tiles = tiles.shape[0] if tiles.ndim == 2 else 0
        self.row_begin = int(cu[0]) if row_begin is None else int(row_begin)
        self.row_end = int(cu[-1]) if row_end is None else int(row_end)

    def struct(self):
        return skr_segs(self.cu.data_ptr(), self.q_pos.data_ptr(), self.k_start.data_ptr(), self.k_len.data_ptr(),
                        self.tiles.data_ptr() if self.n_tiles else 0, self.n_seg, self.n_tiles, self.row_begin,
                        self.row_end)


def make_segs(shape, cu, q_pos, k_start, k_len, kind="fwd", device="cuda", band_rows=None):
    """Host work list (skr_tiles_fwd / skr_tiles_bwd) + device tables for one segment class.
    band_rows (bwd): query-band height of the work items; None = the library's choice for the shape."""
    n = len(cu) - 1
    if kind == "fwd":
        tiles = skr_tiles_fwd(cu, q_pos, n, skr_attn_block_m(shape))
    else:
        band = skr_attn_bwd_band_rows(shape) if band_rows is None else int(band_rows)
        tiles = skr_tiles_bwd(cu, q_pos, k_len, n, skr_attn_block_n(shape), band)
    return DeviceSegs(cu, q_pos, k_start, k_len, tiles, device=device)


def skr_attn_fwd(shape, segs: DeviceSegs, q, k, v, o, lse, stream=None):
    fn = _sig("skr_attn_fwd", i32, P(skr_attn_shape), P(skr_segs), vp, vp, vp, vp, vp, i32, i32, vp)
    g = segs.struct()
    _check(fn(C.byref(shape), C.byref(g), _tptr(q), _tptr(k), _tptr(v), _tptr(o), _tptr(lse), q.shape[0], k.shape[0],
              _stream(stream)))


def skr_attn_bwd(shape, segs: DeviceSegs, q, k, v, o, dout, lse, dq, dk, dv, kv_accumulate, ws, stream=None):
    fn = _sig("skr_attn_bwd", i32, P(skr_attn_shape), P(skr_segs), vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, i32,
              vp, C.c_size_t, vp)
    g = segs.struct()
    _check(fn(C.byref(shape), C.byref(g), _tptr(q), _tptr(k), _tptr(v), _tptr(o), _tptr(dout), _tptr(lse), _tptr(dq),
              _tptr(dk), _tptr(dv), int(kv_accumulate), q.shape[0], k.shape[0], _tptr(ws),
              ws.numel() * ws.element_size(), _stream(stream)))


def skr_attn_bwd_peer(shape, segs: DeviceSegs, q, k, v, o, dout, lse, dq, peer_dk, peer_dv, row_map, pad_rows_P, ws,
                      stream=None):
    """Row f3 step two: backward of the distributed chunks with the dK / dV partials red-added into
    the owners' fp32 accumulators (peer_dk / peer_dv: int64 device tensors of addresses)."""
    fn = _sig("skr_attn_bwd_peer", i32, P(skr_attn_shape), P(skr_segs), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32,
              i32, i32, vp, C.c_size_t, vp)
    g = segs.struct()
    _check(fn(C.byref(shape), C.byref(g), _tptr(q), _tptr(k), _tptr(v), _tptr(o), _tptr(dout), _tptr(lse), _tptr(dq),
              _tptr(peer_dk), _tptr(peer_dv), _tptr(row_map), int(pad_rows_P), q.shape[0], k.shape[0], _tptr(ws),
              ws.numel() * ws.element_size(), _stream(stream)))


def skr_pack_owner_rows(chunk_table, natural_rows):
    """-> int32 [natural_rows]: natural row -> owner * P + row in the owner's distributed prefix."""
    t = np.ascontiguousarray(chunk_table, np.int32).reshape(-1)
    out = np.zeros(max(int(natural_rows), 0), np.int32)
    _check(_sig("skr_pack_owner_rows", i32, P(i32), i32, i32, P(i32))(
        _ptr(t, i32), len(t) // 6, int(natural_rows), _ptr(out, i32)))
    return out


def _rowbytes(t):
    return t[0].numel() * t.element_size() if t.shape[0] else 0


def skr_pack_rows(src, src_row, dst, stream=None):
    fn = _sig("skr_pack_rows", i32, vp, vp, i32, i32, vp, vp)
    _check(fn(_tptr(src), _tptr(src_row), dst.shape[0], dst[0].numel() * dst.element_size() if dst.shape[0] else 16,
              _tptr(dst), _stream(stream)))


def skr_unpack_rows(src, src_row, dst, stream=None):
    fn = _sig("skr_unpack_rows", i32, vp, vp, i32, i32, vp, vp)
    _check(fn(_tptr(src), _tptr(src_row), src.shape[0], src[0].numel() * src.element_size() if src.shape[0] else 16,
              _tptr(dst), _stream(stream)))


def skr_gather_chunks(gathered, chunk_table, n_chunks, natural, stream=None):
    fn = _sig("skr_gather_chunks", i32, vp, vp, i32, i32, vp, vp)
    rb = natural[0].numel() * natural.element_size()
    _check(fn(_tptr(gathered), _tptr(chunk_table), int(n_chunks), rb, _tptr(natural), _stream(stream)))


def skr_scatter_chunks(natural, chunk_table, n_chunks, pad_rows_P, cp, rankmajor, stream=None):
    fn = _sig("skr_scatter_chunks", i32, vp, vp, i32, i32, i32, i32, vp, vp)
    rb = rankmajor[0].numel() * rankmajor.element_size()
    _check(fn(_tptr(natural), _tptr(chunk_table), int(n_chunks), rb, int(pad_rows_P), int(cp), _tptr(rankmajor),
              _stream(stream)))


def skr_cast_f32_bf16(src, dst, stream=None):
    fn = _sig("skr_cast_f32_bf16", i32, vp, vp, i64, vp)
    _check(fn(_tptr(src), _tptr(dst), src.numel(), _stream(stream)))


# ---------------------------------------------------------------------------- row f4: ring CP
def skr_ring_segs(mb_lens, assign, cp, rank, step, cls):
    """Host segment tables of ring hop `step`, key-chunk class `cls` on `rank` (include/skrull.h)."""
    L = np.ascontiguousarray(mb_lens, np.int64)
    A = np.ascontiguousarray(assign, np.int32)
    n = i32()
    fn = _sig("skr_ring_segs", i32, P(i64), P(i32), i32, i32, i32, i32, i32, P(i32), P(i32), P(i32), P(i32), i32,
              P(i32))
    cap = 0
    for _ in range(2):
        cu = np.zeros(cap + 1, np.int32)
        qp, ks, kl = (np.zeros(max(cap, 1), np.int32) for _ in range(3))
        st = fn(_ptr(L, i64), _ptr(A, i32), len(L), int(cp), int(rank), int(step), int(cls), _ptr(cu, i32),
                _ptr(qp, i32), _ptr(ks, i32), _ptr(kl, i32), cap, C.byref(n))
        if st == SKR_OK:
            m = n.value
            return {"cu_seqlens_q": cu[:m + 1], "q_pos": qp[:m], "k_start": ks[:m], "k_len": kl[:m], "n_seg": m}
        if st != SKR_E_CAPACITY:
            _check(st)
        cap = n.value
    raise SkrullError(SKR_E_CAPACITY, "ring segments")


def skr_attn_merge(shape, o_part, lse_part, o_acc, lse_acc, row_begin, row_end, first, stream=None):
    fn = _sig("skr_attn_merge", i32, P(skr_attn_shape), vp, vp, vp, vp, i32, i32, i32, i32, vp)
    _check(fn(C.byref(shape), _tptr(o_part), _tptr(lse_part), _tptr(o_acc), _tptr(lse_acc), int(row_begin),
              int(row_end), lse_acc.shape[-1], int(first), _stream(stream)))


def skr_attn_bwd_acc(shape, segs: DeviceSegs, q, k, v, o, dout, lse, dq, dk, dv, ws, stream=None):
    fn = _sig("skr_attn_bwd_acc", i32, P(skr_attn_shape), P(skr_segs), vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32,
              vp, C.c_size_t, vp)
    g = segs.struct()
    _check(fn(C.byref(shape), C.byref(g), _tptr(q), _tptr(k), _tptr(v), _tptr(o), _tptr(dout), _tptr(lse), _tptr(dq),
              _tptr(dk), _tptr(dv), q.shape[0], k.shape[0], _tptr(ws), ws.numel() * ws.element_size(),
              _stream(stream)))


# ---------------------------------------------------------------------------- a5-a9 composite step
class skr_cp_step(C.Structure):
    _fields_ = [("local_fwd", skr_segs), ("local_bwd", skr_segs), ("dist_fwd", skr_segs), ("dist_bwd", skr_segs),
                ("chunk_table", vp), ("n_chunks", i32), ("cp", i32), ("rows", i32), ("dist_rows", i32),
                ("pad_rows_P", i32), ("natural_rows", i32), ("buf_rows", i32), ("src_row", vp),
                ("q_src", vp), ("k_src", vp), ("v_src", vp), ("do_src", vp),
                ("q", vp), ("k", vp), ("v", vp), ("o", vp), ("dout", vp), ("dq", vp), ("dk", vp), ("dv", vp),
                ("lse", vp), ("k_gathered", vp), ("v_gathered", vp), ("k_natural", vp), ("v_natural", vp),
                ("dk_partial", vp), ("dv_partial", vp), ("dk_rankmajor", vp), ("dv_rankmajor", vp),
                ("dk_reduced", vp), ("dv_reduced", vp), ("ws", vp), ("ws_bytes", C.c_size_t),
                ("timing_events", vp)]


class AttnPlan:
    """skr_attn_plan wrapper (opaque: shape + packed-buffer row capacity)."""

    def __init__(self, shape, max_rows):
        self.h = vp()
        _check(_sig("skr_attn_plan_create", i32, P(skr_attn_shape), i32, P(vp))(C.byref(shape), int(max_rows),
                                                                               C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            _sig("skr_attn_plan_destroy", None, vp)(self.h)
            self.h = vp()


def skr_cp_attn_fwd(comm, plan, step, main=None, side=None):
    _check(_sig("skr_cp_attn_fwd", i32, vp, vp, P(skr_cp_step), vp, vp)(
        comm.h if comm is not None else None, plan.h, C.byref(step), _stream(main), _stream(side)))


def skr_cp_attn_bwd(comm, plan, step, main=None, side=None):
    _check(_sig("skr_cp_attn_bwd", i32, vp, vp, P(skr_cp_step), vp, vp)(
        comm.h if comm is not None else None, plan.h, C.byref(step), _stream(main), _stream(side)))


# ---------------------------------------------------------------------------- f3: peer-memory exchange
def skr_ipc_blob_bytes() -> int:
    return _sig("skr_ipc_blob_bytes", i32)()


def skr_ipc_export(t) -> bytes:
    """IPC blob (handle + offset) of a device tensor's storage start."""
    n = skr_ipc_blob_bytes()
    buf = (C.c_uint8 * n)()
    _check(_sig("skr_ipc_export", i32, vp, vp)(_tptr(t), C.cast(buf, vp)))
    return bytes(buf)


def skr_ipc_import(blob: bytes) -> int:
    """Device address in this process of another process's exported tensor."""
    buf = (C.c_uint8 * len(blob))(*blob)
    out = vp()
    _check(_sig("skr_ipc_import", i32, vp, P(vp))(C.cast(buf, vp), C.byref(out)))
    return int(out.value)


def skr_ipc_close_all():
    _check(_sig("skr_ipc_close_all", i32)())


def skr_peer_gather_chunks(peer_packed, chunk_table, n_chunks, pad_rows_P, natural, stream=None):
    """peer_packed: int64 device tensor [N] of the ranks' packed K (or V) buffer addresses."""
    fn = _sig("skr_peer_gather_chunks", i32, vp, vp, i32, i32, i32, vp, vp)
    rb = natural[0].numel() * natural.element_size()
    _check(fn(_tptr(peer_packed), _tptr(chunk_table), int(n_chunks), rb, int(pad_rows_P), _tptr(natural),
              _stream(stream)))


def skr_peer_reduce_chunks(peer_partials, nranks, rank, chunk_table, n_chunks, row_elems, pad_rows_P, dst,
                           stream=None):
    """peer_partials: int64 device tensor [N] of the ranks' fp32 natural partial buffers; dst bf16 or fp32."""
    import torch
    fn = _sig("skr_peer_reduce_chunks", i32, vp, i32, i32, vp, i32, i32, i32, vp, i32, vp)
    _check(fn(_tptr(peer_partials), int(nranks), int(rank), _tptr(chunk_table), int(n_chunks), int(row_elems),
              int(pad_rows_P), _tptr(dst), 1 if dst.dtype == torch.bfloat16 else 0, _stream(stream)))


def skr_peer_signal(peer_flags, nranks, rank, epoch, stream=None):
    _check(_sig("skr_peer_signal", i32, vp, i32, i32, C.c_uint32, vp)(_tptr(peer_flags), int(nranks), int(rank),
                                                                      int(epoch) & 0xFFFFFFFF, _stream(stream)))


def skr_peer_wait(flags, nranks, epoch, err, stream=None):
    _check(_sig("skr_peer_wait", i32, vp, i32, C.c_uint32, vp, vp)(_tptr(flags), int(nranks), int(epoch) & 0xFFFFFFFF,
                                                                   _tptr(err), _stream(stream)))


class PeerComm:
    """Row f3 exchange context of one CP group: the epoch-flag array every peer writes into, and the
    IPC exchange of buffer addresses over a torch process group (control plane only)."""

    MAX_RANKS = 64

    def __init__(self, nranks, rank, group=None):
        import torch
        self.nranks, self.rank, self.group = nranks, rank, group
        self.flags = torch.zeros(self.MAX_RANKS, dtype=torch.int32, device="cuda")
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.epoch = 0
        torch.cuda.synchronize()
        self.peer_flags = self.exchange([self.flags])[0]

    def exchange(self, tensors):
        """-> one int64 device tensor [nranks] of addresses per input tensor (collective)."""
        import torch
        import torch.distributed as dist
        blobs = [skr_ipc_export(t) for t in tensors]
        allb = [None] * self.nranks
        dist.all_gather_object(allb, blobs, group=self.group)
        out = []
        for i, t in enumerate(tensors):
            addrs = [t.data_ptr() if r == self.rank else skr_ipc_import(allb[r][i]) for r in range(self.nranks)]
            out.append(torch.tensor(addrs, dtype=torch.int64, device="cuda"))
        return out

    def signal(self, stream=None) -> int:
        """Enqueue: this rank reached the next epoch. Returns the epoch to wait for."""
        self.epoch += 1
        skr_peer_signal(self.peer_flags, self.nranks, self.rank, self.epoch, stream)
        return self.epoch

    def wait(self, epoch, stream=None):
        skr_peer_wait(self.flags, self.nranks, epoch, self.err, stream)

    def check(self):
        """Raise if a peer wait timed out since the last check (the error word is then cleared, so
        one timeout is reported once). Call after every synchronize of a step that used the
        exchange: a timed-out wait lets the stream continue on stale peer data."""
        if int(self.err.item()):
            self.err.zero_()
            raise SkrullError(SKR_E_CUDA, "peer exchange: a peer never signalled (10 s); "
                                          "the step's K/V or dK/dV used stale peer data")

    def close(self):
        skr_ipc_close_all()


# ---------------------------------------------------------------------------- CP communicator
class Comm:
    """skr_comm wrapper; the NCCL unique id is broadcast over an existing torch process group."""

    def __init__(self, nranks, rank, group=None, src=0):
        """nranks / rank: the CP group's size and this rank's index in it; `group` the torch process
        group spanning it and `src` the GLOBAL rank of its first member (which draws the NCCL id)."""
        import torch
        import torch.distributed as dist
        n = _sig("skr_nccl_id_bytes", i32)()
        buf = (C.c_uint8 * n)()
        if rank == 0:
            _check(_sig("skr_nccl_get_id", i32, vp)(C.cast(buf, vp)))
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if nranks > 1:
            # an NCCL process group only moves device tensors; gloo takes host tensors
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=src, group=group)
            t = t.cpu()
        buf = (C.c_uint8 * n)(*t.tolist())
        self.h = vp()
        _check(_sig("skr_comm_create", i32, vp, i32, i32, P(vp))(C.cast(buf, vp), int(nranks), int(rank),
                                                                  C.byref(self.h)))
        self.nranks, self.rank = nranks, rank

    def all_gather(self, send, recv, stream=None):
        _check(_sig("skr_comm_all_gather", i32, vp, vp, vp, C.c_size_t, vp)(
            self.h, _tptr(send), _tptr(recv), send.numel() * send.element_size(), _stream(stream)))

    def reduce_scatter_f32(self, send, recv, stream=None):
        _check(_sig("skr_comm_reduce_scatter_f32", i32, vp, vp, vp, C.c_size_t, vp)(
            self.h, _tptr(send), _tptr(recv), recv.numel(), _stream(stream)))

    def all_reduce_f32(self, buf, stream=None):
        _check(_sig("skr_comm_all_reduce_f32", i32, vp, vp, C.c_size_t, vp)(
            self.h, _tptr(buf), buf.numel(), _stream(stream)))

    def ring_shift(self, sends, recvs, stream=None):
        """One ring hop (row f4): sends[i] to rank + 1, rank - 1's into recvs[i] (one NCCL group)."""
        n = len(sends)
        sb = (vp * max(n, 1))(*[_tptr(t) for t in sends])
        rb = (vp * max(n, 1))(*[_tptr(t) for t in recvs])
        nb = (C.c_size_t * max(n, 1))(*[t.numel() * t.element_size() for t in sends])
        _check(_sig("skr_comm_ring_shift", i32, vp, vp, vp, vp, i32, vp)(
            self.h, C.cast(sb, vp), C.cast(rb, vp), C.cast(nb, vp), n, _stream(stream)))

    def size(self):
        """-> (nranks, rank) as the library sees the communicator."""
        n, r = i32(), i32()
        _check(_sig("skr_comm_size", i32, vp, P(i32), P(i32))(self.h, C.byref(n), C.byref(r)))
        return n.value, r.value

    def check(self):
        """Raise SkrullError(SKR_E_NCCL) if NCCL reported an asynchronous error."""
        _check(_sig("skr_comm_async_error", i32, vp)(self.h))

    def wait(self, stream=None, timeout_s=300.0):
        """Host-wait for the work enqueued on `stream`, polling NCCL's asynchronous error state; on
        an error or after timeout_s the communicator is aborted and SkrullError(SKR_E_NCCL) raised
        (a dead peer cannot hang the caller)."""
        _check(_sig("skr_comm_wait", i32, vp, vp, f64)(self.h, _stream(stream), float(timeout_s)))

    def close(self):
        if self.h:
            _sig("skr_comm_destroy", None, vp)(self.h)
            self.h = vp()
