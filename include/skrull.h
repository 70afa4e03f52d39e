/* skrull.h -- C ABI of libskrull.so: the B200-native hot path of Skrull (arXiv 2505.19609).
 *
 * Citations: P:n = line n of PAPER.md (the paper's LaTeX), S:n = line n of SPEC.md,
 * R# = a reading in DESIGN.md's ambiguity ledger.
 *
 * Conventions (all entry points)
 *  - Every function returning skr_status never throws, aborts or exits. On failure it returns a
 *    non-zero status and skr_last_error() holds a thread-local message.
 *  - The caller allocates ALL outputs (host and device) and owns them; sizes come from the
 *    *_bounds / *_ws_bytes queries. The library keeps no pointer past the call, except inside
 *    explicit opaque objects (skr_comm) with create/destroy pairs.
 *  - Host functions are pure and re-entrant. Device functions enqueue work on the caller's
 *    stream(s) and return without synchronising; errors of the enqueued work surface at the
 *    caller's next synchronisation (launch errors are returned as SKR_E_CUDA immediately).
 *  - Device entry points require an sm_100a GPU (B200); on anything else they return
 *    SKR_E_UNSUPPORTED. There is no CPU fallback.
 *  - Integers: sequence lengths int64; row indices and table entries int32 (a packed rank
 *    buffer holds < 2^31 rows).
 */
#ifndef SKRULL_H_
#define SKRULL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t skr_status;
enum {
  SKR_OK = 0,
  SKR_E_ARG = 1,         /* bad argument (null pointer, negative size, inconsistent shape) */
  SKR_E_SCHEDULE = 2,    /* Alg. 1 Assert: roll-back impossible, or disabled (Table 3 "OOM") */
  SKR_E_GDS = 3,         /* Alg. 2: no init <= |Subset|+1 feasible (R15) */
  SKR_E_BUDGET = 4,      /* Memory(S) budget <= beta (Appendix C.1) */
  SKR_E_PROFILE = 5,     /* fewer than 2 profile points at/above the threshold */
  SKR_E_OVERFLOW = 6,    /* exact integer FLOPs / scaled ledgers would overflow int64 */
  SKR_E_CAPACITY = 7,    /* caller buffer too small */
  SKR_E_CUDA = 8,        /* CUDA launch / runtime error */
  SKR_E_NCCL = 9,        /* NCCL error */
  SKR_E_UNSUPPORTED = 10 /* no sm_100a device, or shape outside the kernels' support */
};

const char* skr_status_string(skr_status s);
const char* skr_last_error(void);
int32_t skr_abi_version(void); /* bumps on any signature change */

/* ------------------------------------------------------------------ a1: cost model
 * Appendix C. */
typedef struct {
  int64_t hidden;     /* h   = Hq * d */
  int64_t kv_hidden;  /* h_kv = Hkv * d */
  int64_t pack_batch; /* b, 1 with sequence packing */
} skr_model;
typedef struct {
  double slope;     /* alpha */
  double intercept; /* beta / T_fixed */
} skr_fit;
typedef struct {
  skr_fit comp;          /* Eq. 13: T_comp = alpha FLOPs + beta */
  skr_fit comm;          /* Eq. 15: T_comm = alpha V + T_fixed, 0 when V == 0    (R26) */
  skr_fit mem;           /* Memory(S) = alpha S + beta */
  double bytes_per_elem; /* V is Eq. 14 elements x bytes_per_elem              (R25) */
  double dist_penalty;   /* multiplies T_comp(Dist); 1 = Eq. 2 exactly  */
} skr_cost;
typedef struct {
  int32_t cp;            /* N, CP degree */
  int32_t dp;            /* ws, DP degree */
  int64_t bucket_tokens; /* C, BucketSize per rank */
  int32_t rollback;      /* 1 = Alg. 3 RollBack enabled; 0 reproduces Table 3's "w/o" rows */
} skr_cluster;

/* Eq. 12: FLOPs(S) = 20 b h^2 S + 4 b h h_kv S + 4 b h S^2, exact. SKR_E_OVERFLOW past int64. */
skr_status skr_flops(int64_t S, const skr_model* m, int64_t* out);
/* Eq. 14: Volume(S) = b S h_kv elements. */
skr_status skr_volume(int64_t S, const skr_model* m, int64_t* out);
/* Eq. 13; zero FLOPs cost zero (R36). */
double skr_t_comp(double flops, const skr_fit* fit);
/* Eq. 15; 0 when volume == 0 (R26). */
double skr_t_comm(double volume, const skr_fit* fit);
/* Least squares over points with x >= min_x; negative intercept clamped to 0.
 * SKR_E_PROFILE with < 2 qualifying points. */
skr_status skr_fit_linear(const double* x, const double* y, int32_t n, double min_x, skr_fit* out);
/* C = floor((budget - beta) / alpha); SKR_E_BUDGET if budget <= beta. */
skr_status skr_bucket_size(double budget, const skr_fit* mem, int64_t* C);

/* ------------------------------------------------------------------ a2/a3: schedulers */
/* Alg. 1 + Alg. 3 (readings R1-R10). `lens[K]` in input order; writes
 * assign[K] in input order: -1 = distributed, v in [0,cp) = local on CP rank v.
 * Exact integer ledgers scaled by N (R4). On SKR_E_SCHEDULE, *fail_idx = sorted position of the
 * sequence that could not be placed. n_rollbacks / fail_idx may be NULL. */
skr_status skr_dacp(const int64_t* lens, int32_t K, const skr_cluster* cl, const skr_model* m, int32_t* assign,
                    int32_t* n_rollbacks, int32_t* fail_idx);
/* Eq. 1-7 for a given assignment. per_rank_time[cp] (may be NULL); an infeasible
 * plan (Eq. 7) is still evaluated with *feasible = 0. */
skr_status skr_eval_tdacp(const int64_t* lens, const int32_t* assign, int32_t K, const skr_cluster* cl,
                          const skr_model* m, const skr_cost* cost, double* per_rank_time, double* comm_time,
                          double* dist_time, double* tdacp, int32_t* feasible);
/* Alg. 2 line 1 "Binpack(ws, FLOPs(S[K]))" as greedy LPT (R16). bin_of_seq[K]. */
skr_status skr_lpt(const int64_t* lens, int32_t K, int32_t bins, const skr_model* m, int32_t* bin_of_seq);
/* Alg. 2 (R11-R15) for DP rank `dp_rank`: mb_of_seq[K] = micro-batch index of each
 * sequence of this rank's LPT bin, -1 for sequences of other DP ranks. */
skr_status skr_gds(const int64_t* lens, int32_t K, const skr_cluster* cl, const skr_model* m, int32_t dp_rank,
                   int32_t* mb_of_seq, int32_t* n_mb);
/* Whole-iteration plan: LPT over cl->dp ranks, GDS per rank, DACP per micro-batch.
 * dp_of_seq[K], mb_of_seq[K], assign[K] (DACP result inside its micro-batch), n_mb_per_dp[cl->dp].
 * Every rank computes the identical plan with no communication. */
skr_status skr_plan(const int64_t* lens, int32_t K, const skr_cluster* cl, const skr_model* m, int32_t* dp_of_seq,
                    int32_t* mb_of_seq, int32_t* assign, int32_t* n_mb_per_dp, int32_t* n_rollbacks);

/* Baselines (row f1): Alg. 4 round-robin (R27: input order, shard by N, R6 roll-back on
 * RemainBucket) -> assign[K] as skr_dacp; and the DeepSpeed-like full-shard plan (S:398-406, P:101,
 * P:316): FIFO micro-batches under C*N tokens (mb_of_seq[K], n_mb), every sequence distributed. */
skr_status skr_round_robin(const int64_t* lens, int32_t K, const skr_cluster* cl, int32_t* assign,
                           int32_t* n_rollbacks, int32_t* fail_idx);
skr_status skr_full_shard(const int64_t* lens, int32_t K, const skr_cluster* cl, int32_t* mb_of_seq, int32_t* n_mb);

/* ------------------------------------------------------------------ a4: packer (host)
 * One micro-batch (mb_lens[K_mb] in micro-batch input order, its DACP assign), CP rank `rank`.
 * Layout (R20-R23): zigzag chunks c of 2N, [floor(cS/2N), floor((c+1)S/2N)), rank j owns j and
 * 2N-1-j; packed rows = [distributed chunks, sequences ascending (length, index), chunk j then
 * 2N-1-j] ++ [locals on j, ascending]. Source order ("rank-natural"): this rank's rows in input
 * order, positions ascending. */
skr_status skr_pack_bounds(const int64_t* mb_lens, const int32_t* assign, int32_t K_mb, int32_t cp, int32_t rank,
                           int32_t* n_seg, int32_t* n_dist_seg, int32_t* n_rows, int32_t* dist_rows,
                           int32_t* pad_rows_P, int32_t* natural_rows, int32_t* n_chunks);
/* Writes cu_seqlens_q[n_seg+1], q_pos/k_start/k_len/seg_seq/seg_chunk[n_seg], src_row[n_rows].
 * k_start: packed row of the segment (locals) or row in the natural distributed-K/V buffer
 * (distributed). k_len = q_pos + q_len (bottom-right causal). */
skr_status skr_pack_rank(const int64_t* mb_lens, const int32_t* assign, int32_t K_mb, int32_t cp, int32_t rank,
                         int32_t* cu_seqlens_q, int32_t* q_pos, int32_t* k_start, int32_t* k_len, int32_t* seg_seq,
                         int32_t* seg_chunk, int32_t* src_row);
/* Chunk table of all distributed sequences (the same on every rank): n_chunks rows of 6 int32:
 * {seq, chunk, owner, gathered_row (owner*P + offset in owner's prefix), natural_row, len}. */
skr_status skr_pack_chunks(const int64_t* mb_lens, const int32_t* assign, int32_t K_mb, int32_t cp,
                           int32_t* chunk_table);
/* Attention work lists (host; the caller owns `tiles`, cap_tiles = its capacity in items; on
 * SKR_E_CAPACITY *n_tiles is the number needed).
 * fwd: pairs {segment, query tile} of block_m rows, ordered longest-work-first (LPT).
 * bwd: quadruples {segment, key tile, q_lo, q_hi}: key tile t of block_n keys over [0, k_len) with the
 *   segment-relative query rows [q_lo, q_hi) it processes (only those that also see the tile, i.e.
 *   query position >= key position). band_rows = 0, or a segment of at most band_rows queries: one
 *   item per key tile, q_lo = 0, q_hi = q_len. Longer segments are split into query bands
 *   [b*band_rows, (b+1)*band_rows) (band_rows a multiple of 128), one item per (key tile, band) that
 *   holds a visible query; these come first, segment by segment and band by band with key tiles
 *   ascending (the CTAs in flight share one band's Q / dO / dQ rows in L2), then the rest in LPT
 *   order. skr_attn_bwd sums the bands' dK / dV partials (fp32) before writing dK / dV. */
skr_status skr_tiles_fwd(const int32_t* cu_seqlens_q, const int32_t* q_pos, int32_t n_seg, int32_t block_m,
                         int32_t* tiles, int32_t cap_tiles, int32_t* n_tiles);
skr_status skr_tiles_bwd(const int32_t* cu_seqlens_q, const int32_t* q_pos, const int32_t* k_len, int32_t n_seg,
                         int32_t block_n, int32_t band_rows, int32_t* tiles, int32_t cap_tiles, int32_t* n_tiles);

/* ------------------------------------------------------------------ a5-a9: device
 * All pointers below are DEVICE pointers; `stream` is a cudaStream_t passed as void*. */
enum { SKR_BF16 = 0, SKR_FP32 = 1 };
typedef struct {
  int32_t hq, hkv, d; /* q heads, kv heads (hq % hkv == 0, GQA groups contiguous, R30), head dim */
  int32_t dtype;      /* SKR_BF16: tcgen05 kernels (d in {64,128}); SKR_FP32: fp32 test mode (R31) */
  float scale;        /* softmax scale, 1/sqrt(d) (R29) */
} skr_attn_shape;
typedef struct {                /* one segment class (locals, or distributed chunks) of one rank */
  const int32_t* cu_seqlens_q;  /* [n_seg+1] packed query rows */
  const int32_t* q_pos;         /* [n_seg] position of the first query in its sequence */
  const int32_t* k_start;       /* [n_seg] first row of the segment's keys in the K/V buffer */
  const int32_t* k_len;         /* [n_seg] keys: query i sees keys j < min(k_len, q_pos + i + 1); q_pos + q_len
                                   for a whole causal segment, less for a ring-CP key chunk (0: none) */
  const int32_t* tiles;         /* work list: [2*n_tiles] from skr_tiles_fwd, [4*n_tiles] from skr_tiles_bwd */
  int32_t n_seg, n_tiles;
  int32_t row_begin, row_end;   /* host ints: the class's packed query rows are [row_begin, row_end) */
} skr_segs;

/* Input contract of the attention calls: every row of q / k / v (and dout) inside
 * [0, n_q_rows) / [0, n_kv_rows) must be finite, also rows no segment owns -- a 128-row tile reads
 * past a segment's end and the tensor cores multiply those rows by exact zeros (0 x NaN = NaN).
 * Forward (row a7; Eq. 2-4): per segment and q-head h (kv head h*hkv/hq),
 * O = softmax(scale QK^T + bottom-right causal mask) V, LSE = natural-log row logsumexp; keys at or
 * past k_len are masked too, and a query that sees no key gets O = 0, LSE = -inf (ring CP partials).
 * q, o: [n_q_rows][hq][d]; k, v: [n_kv_rows][hkv][d]; lse: fp32 [hq][n_q_rows].
 * bf16 in/out with fp32 accumulation (SKR_BF16) or fp32 throughout (SKR_FP32).
 * `tiles` must come from skr_tiles_fwd with block_m = skr_attn_block_m(shape): 128 query rows
 * (bf16), 32 (fp32), or 256 for d = 128 in the CTA-pair forward variant library
 * (libskrull_fwd2sm.so, built with -DSKR_FWD_2SM_BUILD; fixed per library build, never switched at run time). */
int32_t skr_attn_block_m(const skr_attn_shape* s);
int32_t skr_attn_block_n(const skr_attn_shape* s);
/* The library's query-band height for skr_tiles_bwd (0 = no bands) for this shape. */
int32_t skr_attn_bwd_band_rows(const skr_attn_shape* s);
skr_status skr_attn_fwd(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k, const void* v,
                        void* o, float* lse, int32_t n_q_rows, int32_t n_kv_rows, void* stream);
/* Backward (row a8): D = rowsum(dO o O); dQ, dK, dV of the plain definition.
 * dq: [n_q_rows][hq][d] written for the segments' rows (bf16 / fp32 per dtype).
 * kv_accumulate = 0: dk, dv [n_kv_rows][hkv][d] of dtype are WRITTEN for the segments' key rows
 *   (locals: each key row belongs to exactly one segment).
 * kv_accumulate = 1: dk, dv are fp32 [n_kv_rows][hkv][d] and are ADDED to (distributed chunks of one
 *   sequence share key rows; the caller zeroes them once).
 * ws: fp32 scratch of skr_attn_bwd_ws_bytes(s, n_q_rows): the D rows, the fp32 dQ accumulator and
 *   (kv_accumulate = 0 with query-banded work items) fp32 dK / dV band accumulators indexed by key row,
 *   which is why kv_accumulate = 0 requires n_kv_rows <= n_q_rows (SKR_E_ARG otherwise; for local
 *   segments the K / V rows are the packed query rows). `tiles` from skr_tiles_bwd with block_n =
 *   skr_attn_block_n. */
size_t skr_attn_bwd_ws_bytes(const skr_attn_shape* s, int32_t n_q_rows);
skr_status skr_attn_bwd(const skr_attn_shape* s, const skr_segs* g, const void* q,
                        const void* k, const void* v, const void* o, const void* dout, const float* lse, void* dq,
                        void* dk, void* dv, int32_t kv_accumulate, int32_t n_q_rows, int32_t n_kv_rows, void* ws,
                        size_t ws_bytes, void* stream);

/* a5 pack: dst[r] = src[src_row[r]] for n_rows rows of row_bytes (multiple of 16). */
skr_status skr_pack_rows(const void* src, const int32_t* src_row, int32_t n_rows, int32_t row_bytes, void* dst,
                         void* stream);
/* a5 inverse: dst[src_row[r]] = src[r]. */
skr_status skr_unpack_rows(const void* src, const int32_t* src_row, int32_t n_rows, int32_t row_bytes, void* dst,
                           void* stream);
/* a6 reorder: gathered [N][P] rank-major rows -> natural distributed order, via the chunk table. */
skr_status skr_gather_chunks(const void* gathered, const int32_t* chunk_table, int32_t n_chunks, int32_t row_bytes,
                             void* natural, void* stream);
/* a9 permute: natural fp32 partials -> rank-major [N][P] rows. chunk_table must be skr_pack_chunks'
 * (2N rows per distributed sequence, else SKR_E_ARG); the same launch zeroes exactly the padding
 * rows of each rank slot (beyond the rank's own distributed rows: the reduce-scatter sums them). */
skr_status skr_scatter_chunks(const void* natural, const int32_t* chunk_table, int32_t n_chunks, int32_t row_bytes,
                              int32_t pad_rows_P, int32_t cp, void* rankmajor, void* stream);
/* a9 cast: fp32 -> bf16, n elements. */
skr_status skr_cast_f32_bf16(const float* src, void* dst, int64_t n, void* stream);

/* Row f3 (first step): the CP exchange over peer memory instead of NCCL collectives
 * (P:122 names the all-gather / its mirror, P:57 leaves the CP method open).
 * Buffers of the other ranks of the CP group are mapped with CUDA IPC; on NVLink / NVSwitch the
 * kernels' loads and stores are peer accesses. All pointer arrays are DEVICE arrays of nranks
 * uint64 device addresses (this rank's own buffer at index rank). */
int32_t skr_ipc_blob_bytes(void); /* size of an export blob: IPC handle + offset in its allocation */
/* Export a device pointer (may point inside a larger cudaMalloc allocation) for another process. */
skr_status skr_ipc_export(const void* dev_ptr, void* blob_out);
/* Map another process's exported pointer (one mapping per allocation per process, refcounted);
 * SKR_E_CUDA if the handle cannot be opened (e.g. the same process that exported it). */
skr_status skr_ipc_import(const void* blob, void** dev_ptr_out);
skr_status skr_ipc_close_all(void); /* unmap every imported allocation */
/* a6 as one pass: for each chunk-table row, len rows of row_bytes from
 * peer_packed[owner] + (gathered_row - owner*pad_rows_P) rows  ->  natural + natural_row rows.
 * Replaces all-gather + skr_gather_chunks (no [N][P] staging buffer). */
skr_status skr_peer_gather_chunks(const uint64_t* peer_packed, const int32_t* chunk_table, int32_t n_chunks,
                                  int32_t row_bytes, int32_t pad_rows_P, void* natural, void* stream);
/* a9 as one pass: for each chunk OWNED by `rank`, dst row (gathered_row - rank*pad_rows_P + r) =
 * sum over ranks 0..nranks-1 (fixed order) of peer_partials[rank'] fp32 row (natural_row + r),
 * row_elems fp32 per row; dst bf16 (round to nearest even) if dst_bf16, else fp32.
 * Replaces skr_scatter_chunks + reduce-scatter + skr_cast_f32_bf16. */
skr_status skr_peer_reduce_chunks(const uint64_t* peer_partials, int32_t nranks, int32_t rank,
                                  const int32_t* chunk_table, int32_t n_chunks, int32_t row_elems,
                                  int32_t pad_rows_P, void* dst, int32_t dst_bf16, void* stream);
/* Row f3, step two: the a9 reduction fused into the backward of the DISTRIBUTED chunks (a8), so the
 * tensor-core kernel itself performs the collective's data movement: every dK / dV fp32 partial row
 * the kernel produces is red-added (red.global.add.f32, peer stores over NVLink) straight into the
 * accumulator of the rank that OWNS that key row -- no local partial buffer, no permute, no
 * reduce-scatter, no peer-reduce pass. Arguments as skr_attn_bwd for the distributed segment class
 * (k, v = the natural distributed K / V buffer, dq as there), plus:
 *   peer_dk, peer_dv : device arrays [nranks] of the ranks' fp32 accumulators [pad_rows_P][hkv][d]
 *                      (row r = row r of the owner's distributed prefix), zeroed by their owners and
 *                      made visible (epoch flags) before the launch;
 *   row_map          : device int32 [natural rows]: natural row -> owner * pad_rows_P + prefix row
 *                      (skr_pack_owner_rows).
 * The owner casts its accumulator rows [0, dist_rows) into its packed bf16 dK / dV prefix after every
 * rank's kernel has completed (epoch flags). fp32 test mode: the same with atomicAdd. */
skr_status skr_attn_bwd_peer(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k, const void* v,
                             const void* o, const void* dout, const float* lse, void* dq, const uint64_t* peer_dk,
                             const uint64_t* peer_dv, const int32_t* row_map, int32_t pad_rows_P, int32_t n_q_rows,
                             int32_t n_kv_rows, void* ws, size_t ws_bytes, void* stream);
/* Host: row_map for skr_attn_bwd_peer from skr_pack_chunks' table: for every chunk row and r < len,
 * row_map[natural_row + r] = gathered_row + r (= owner * P + row in the owner's distributed prefix).
 * row_map has natural_rows entries; SKR_E_ARG if a chunk row falls outside it. */
skr_status skr_pack_owner_rows(const int32_t* chunk_table, int32_t n_chunks, int32_t natural_rows, int32_t* row_map);
/* Epoch flags (uint32 per rank): signal stores `epoch` into slot `rank` of every peer's flag array
 * (system-scope release after a system fence, ordered after this stream's earlier work); wait
 * blocks the stream until every slot of this rank's flags reached `epoch`, or sets *err = 1 after
 * ~10 s (a peer never signalled) instead of hanging; the stream then continues on stale peer data,
 * so the caller must read *err after synchronising (and clear it) before trusting the step. */
skr_status skr_peer_signal(const uint64_t* peer_flags, int32_t nranks, int32_t rank, uint32_t epoch, void* stream);
skr_status skr_peer_wait(const uint32_t* flags, int32_t nranks, uint32_t epoch, int32_t* err, void* stream);

/* CP communicator (rows a6/a9; NCCL inside the CP group over NVLink/NVSwitch). */
typedef struct skr_comm skr_comm;
int32_t skr_nccl_id_bytes(void); /* size of the unique id blob (128) */
skr_status skr_nccl_get_id(void* id_out);
skr_status skr_comm_create(const void* nccl_id, int32_t nranks, int32_t rank, skr_comm** out);
void skr_comm_destroy(skr_comm* c);
skr_status skr_comm_all_gather(skr_comm* c, const void* send, void* recv, size_t bytes_per_rank, void* stream);
skr_status skr_comm_reduce_scatter_f32(skr_comm* c, const float* send, float* recv, size_t count_per_rank,
                                       void* stream);
skr_status skr_comm_all_reduce_f32(skr_comm* c, float* buf, size_t count, void* stream);
/* Size and this rank's index of the communicator. */
skr_status skr_comm_size(const skr_comm* c, int32_t* nranks, int32_t* rank);
/* SKR_E_NCCL if the communicator reported an asynchronous error (ncclCommGetAsyncError) or was aborted. */
skr_status skr_comm_async_error(skr_comm* c);
/* Failure detection: block the HOST until the work enqueued on `stream` so far has
 * finished, polling the communicator's asynchronous error state; on an NCCL error, or if the work is
 * not done after timeout_s seconds (a dead or stalled peer), abort the communicator (releasing NCCL
 * kernels blocked on the peer) and return SKR_E_NCCL. An aborted communicator rejects further use;
 * skr_comm_destroy still frees it. */
skr_status skr_comm_wait(skr_comm* c, void* stream, double timeout_s);

/* ------------------------------------------------------------------ row f4: ring CP
 * The alternative exchange for distributed sequences (ring attention is one of the CP methods
 * DACP is orthogonal to): instead of all-gathering K/V (R19), each rank's distributed K/V prefix
 * travels N-1 hops along the ring (skr_comm_ring_shift, point-to-point), and at every hop the rank
 * computes its own query chunks against the visiting chunk pair as two partial attentions (one per
 * key chunk of the pair), merged into a running (O, LSE). The backward sends the visiting K/V back
 * around with fp32 dK/dV accumulators that collect every rank's contribution and arrive home after
 * N hops; dQ accumulates in fp32 over the hops. Same plans, same packed layout, same kernels.
 *
 * Host: segments of ring hop `step` (0..N-1) on `rank` for key-chunk class `cls` (0: chunk s,
 * 1: chunk 2N-1-s of the visiting pair from rank s = (rank - step) mod N): one segment per own
 * query chunk in packed-prefix order (cu_seqlens_q covers the rank's dist_rows); k_start indexes
 * rank s's packed prefix; a key chunk before the query chunk is visible whole (q_pos = its length),
 * the own chunk is the causal diagonal (q_pos = 0), a later chunk gets k_len = 0 (no visible key).
 * cap = capacity of q_pos / k_start / k_len (2 * number of distributed sequences needed; cu_seqlens_q
 * holds cap + 1); SKR_E_CAPACITY sets *n_seg to the need. */
skr_status skr_ring_segs(const int64_t* mb_lens, const int32_t* assign, int32_t K_mb, int32_t cp, int32_t rank,
                         int32_t step, int32_t cls, int32_t* cu_seqlens_q, int32_t* q_pos, int32_t* k_start,
                         int32_t* k_len, int32_t cap, int32_t* n_seg);
/* Device: merge a partial attention result into the running one, rows [row_begin, row_end), every
 * q-head: L = log(e^lse_acc + e^lse_part); o_acc = o_acc e^(lse_acc-L) + o_part e^(lse_part-L);
 * lse_acc = L. o_part: [rows][hq][d] of the shape's dtype (a skr_attn_fwd output); o_acc fp32, same
 * layout; lse_*: fp32 [hq][ld_lse], natural log; -inf = empty partial (weight 0). first = 1
 * initialises the running result with the partial. */
skr_status skr_attn_merge(const skr_attn_shape* s, const void* o_part, const float* lse_part, float* o_acc,
                          float* lse_acc, int32_t row_begin, int32_t row_end, int32_t ld_lse, int32_t first,
                          void* stream);
/* Device: backward of one segment class with every gradient an fp32 accumulator the caller owns and
 * zeroes: dq [n_q_rows][hq][d], dk / dv [n_kv_rows][hkv][d] are ADDED to (o / lse: the merged final
 * forward results). Otherwise as skr_attn_bwd. */
skr_status skr_attn_bwd_acc(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k, const void* v,
                            const void* o, const void* dout, const float* lse, float* dq, float* dk, float* dv,
                            int32_t n_q_rows, int32_t n_kv_rows, void* ws, size_t ws_bytes, void* stream);
/* One ring hop: send_bufs[i] (bytes[i]) to rank + 1, receive rank - 1's into recv_bufs[i], one NCCL
 * group on `stream` (a 1-rank communicator sends to itself). */
skr_status skr_comm_ring_shift(skr_comm* c, const void* const* send_bufs, void* const* recv_bufs,
                               const size_t* bytes, int32_t n_bufs, void* stream);

/* ------------------------------------------------------------------ a5-a9 as one call per direction
 * The CP-rank step of one micro-batch (Eq. 2, mirrored for the
 * backward, reading R24), sequenced on a main and a side stream:
 *  fwd: main packs Q/K/V; side all-gathers the K/V distributed prefix (NCCL, CP group) and reorders
 *       it to natural order; main runs the LOCAL tiles meanwhile, then waits and runs the DISTRIBUTED
 *       chunks.
 *  bwd: main packs dO, zeroes the fp32 partials and runs the DISTRIBUTED chunks; side permutes,
 *       reduce-scatters (sum) and casts into the packed dK/dV prefix while main runs the LOCAL tiles;
 *       main then waits for the side stream (the call returns with all work ordered on `main`).
 * With natural_rows == 0 no collective is issued and `comm` may be null. All buffers are caller-owned
 * device memory laid out as DESIGN.md §2 describes; the tables come from skr_pack_rank /
 * skr_pack_chunks / skr_tiles_*. */
typedef struct skr_attn_plan skr_attn_plan;   /* opaque: shape + packed-buffer row capacity */
skr_status skr_attn_plan_create(const skr_attn_shape* s, int32_t max_rows, skr_attn_plan** out);
void skr_attn_plan_destroy(skr_attn_plan* p);
typedef struct {
  skr_segs local_fwd, local_bwd, dist_fwd, dist_bwd; /* segment classes with their work lists */
  const int32_t* chunk_table;   /* [n_chunks * 6] (skr_pack_chunks), device */
  int32_t n_chunks;
  int32_t cp;                   /* CP group size N */
  int32_t rows;                 /* packed rows of this rank */
  int32_t dist_rows;            /* rows of the distributed prefix (all-gather send rows) */
  int32_t pad_rows_P;           /* P = max over ranks of dist_rows (R22) */
  int32_t natural_rows;         /* rows of the natural distributed-K/V buffer */
  int32_t buf_rows;             /* rows allocated in q/k/v/o/dout/dq/dk/dv/lse (>= max(rows, P)) */
  const int32_t* src_row;       /* [rows] packed row -> rank-natural input row (skr_pack_rank) */
  const void *q_src, *k_src, *v_src, *do_src;     /* rank-natural inputs */
  void *q, *k, *v, *o, *dout, *dq, *dk, *dv;      /* packed, [buf_rows][h][d]; rows [rows, buf_rows)
                                                     must hold FINITE values (e.g. zeros): attention
                                                     tiles read them and multiply them by exact zeros */
  float* lse;                                     /* [hq][buf_rows] */
  void *k_gathered, *v_gathered;                  /* [cp*P][hkv][d] */
  void *k_natural, *v_natural;                    /* [natural_rows][hkv][d], kept from fwd to bwd */
  float *dk_partial, *dv_partial;                 /* [natural_rows][hkv][d] fp32 */
  float *dk_rankmajor, *dv_rankmajor;             /* [cp*P][hkv][d] fp32 (reduce-scatter input) */
  float *dk_reduced, *dv_reduced;                 /* [P][hkv][d] fp32 (reduce-scatter output) */
  void* ws;                                       /* skr_attn_bwd workspace for buf_rows */
  size_t ws_bytes;
  void* const* timing_events;   /* optional (NULL: none): 8 caller-created cudaEvent_t recorded on
                                   the main stream around the attention calls (row a10 per-kernel
                                   timing inside the step): fwd [0] before / [1] after the LOCAL
                                   call, [2] before (after the exchange wait) / [3] after the
                                   DISTRIBUTED call; bwd [4] / [5] DISTRIBUTED, [6] / [7] LOCAL. The
                                   events of a call that is skipped are recorded back to back. */
} skr_cp_step;
skr_status skr_cp_attn_fwd(skr_comm* comm, const skr_attn_plan* plan, const skr_cp_step* step, void* main_stream,
                           void* side_stream);
skr_status skr_cp_attn_bwd(skr_comm* comm, const skr_attn_plan* plan, const skr_cp_step* step, void* main_stream,
                           void* side_stream);

/* ------------------------------------------------------------------ diagnostics */
/* UMMA/TMA/TMEM building-block self-test: C[128][n] fp32 from bf16 A/B with operand layout
 * `variant` (0: A K-major, B K-major; 1: B MN-major; 2: A and B MN-major; 3: A written by threads
 * into swizzled smem; 4: A written by threads into TMEM, MMA A operand from TMEM). n in {64,128}, K = 128. */
skr_status skr_selftest_umma(int32_t variant, int32_t n, const void* A, const void* B, float* C, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKRULL_H_ */
