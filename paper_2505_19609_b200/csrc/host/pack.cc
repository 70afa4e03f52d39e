// a4: plan-driven packer tables for one micro-batch and CP rank (readings R20-R23), and the
// LPT-ordered attention work lists.
//
// PAPER.md fixes that a distributed sequence puts S/N tokens on each of the N CP ranks (Eq. 4/7,
// P:158/P:161), that packing removes padding and that the CP exchange is orthogonal to
// DACP. Layout chosen here: zigzag 2N chunks so each rank gets Dist/N causal
// work (Eq. 4), distributed chunks first so the all-gather send buffer is a contiguous prefix.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../common.h"

namespace {

struct Chunk {
  int64_t a, b;  // [a, b) positions
};

inline Chunk chunk_of(int64_t S, int32_t c, int32_t N) {   // R20
  return {(int64_t)c * S / (2 * N), (int64_t)(c + 1) * S / (2 * N)};
}
inline int32_t owner_of(int32_t c, int32_t N) { return c < N ? c : 2 * N - 1 - c; }

struct MbView {
  std::vector<int32_t> order;   // ascending (len, index)
  std::vector<int32_t> dist;    // distributed, in order
  std::vector<int64_t> nat_base;
  int64_t natural_rows = 0;
};

skr_status view(const int64_t* L, const int32_t* A, int32_t K, int32_t N, MbView* v) {
  if (K < 0 || N < 1 || (K > 0 && (!L || !A))) return skr::fail(SKR_E_ARG, "pack: bad arguments");
  v->order.resize(K);
  std::iota(v->order.begin(), v->order.end(), 0);
  std::sort(v->order.begin(), v->order.end(),
            [&](int32_t a, int32_t b) { return L[a] != L[b] ? L[a] < L[b] : a < b; });
  v->nat_base.assign(K, -1);
  for (int32_t k : v->order) {
    if (L[k] < 0) return skr::fail(SKR_E_ARG, "pack: negative length");
    if (A[k] < -1 || A[k] >= N) return skr::fail(SKR_E_ARG, "pack: assign[%d]=%d out of range", k, A[k]);
    if (A[k] == -1) {
      v->dist.push_back(k);
      v->nat_base[k] = v->natural_rows;
      v->natural_rows += L[k];
    }
  }
  if (v->natural_rows > INT32_MAX) return skr::fail(SKR_E_OVERFLOW, "pack: > 2^31 rows");
  return SKR_OK;
}

int64_t dist_rows_of(const int64_t* L, const MbView& v, int32_t N, int32_t j) {
  int64_t r = 0;
  for (int32_t k : v.dist) {
    Chunk x = chunk_of(L[k], j, N), y = chunk_of(L[k], 2 * N - 1 - j, N);
    r += (x.b - x.a) + (y.b - y.a);
  }
  return r;
}

}  // namespace

using skr::fail;

SKR_EXPORT skr_status skr_pack_bounds(const int64_t* L, const int32_t* A, int32_t K, int32_t N, int32_t j,
                                      int32_t* n_seg, int32_t* n_dist_seg, int32_t* n_rows, int32_t* dist_rows,
                                      int32_t* pad_rows_P, int32_t* natural_rows, int32_t* n_chunks) {
  SKR_REQUIRE(N >= 1 && j >= 0 && j < N, "skr_pack_bounds: rank %d out of [0,%d)", j, N);
  MbView v;
  if (skr_status s = view(L, A, K, N, &v)) return s;
  int64_t nloc = 0, rows_loc = 0, P = 0;
  for (int32_t k = 0; k < K; ++k)
    if (A[k] == j) ++nloc, rows_loc += L[k];
  for (int32_t r = 0; r < N; ++r) P = std::max(P, dist_rows_of(L, v, N, r));
  const int64_t dr = dist_rows_of(L, v, N, j);
  if (dr + rows_loc > INT32_MAX || P * N > INT32_MAX) return fail(SKR_E_OVERFLOW, "pack: > 2^31 rows");
  if (n_seg) *n_seg = (int32_t)(2 * v.dist.size() + nloc);
  if (n_dist_seg) *n_dist_seg = (int32_t)(2 * v.dist.size());
  if (n_rows) *n_rows = (int32_t)(dr + rows_loc);
  if (dist_rows) *dist_rows = (int32_t)dr;
  if (pad_rows_P) *pad_rows_P = (int32_t)P;
  if (natural_rows) *natural_rows = (int32_t)v.natural_rows;
  if (n_chunks) *n_chunks = (int32_t)(2 * N * v.dist.size());
  return SKR_OK;
}

SKR_EXPORT skr_status skr_pack_rank(const int64_t* L, const int32_t* A, int32_t K, int32_t N, int32_t j,
                                    int32_t* cu_seqlens_q, int32_t* q_pos, int32_t* k_start, int32_t* k_len,
                                    int32_t* seg_seq, int32_t* seg_chunk, int32_t* src_row) {
  SKR_REQUIRE(N >= 1 && j >= 0 && j < N, "skr_pack_rank: rank out of range");
  SKR_REQUIRE(cu_seqlens_q && q_pos && k_start && k_len && seg_seq && seg_chunk && src_row,
              "skr_pack_rank: null output");
  MbView v;
  if (skr_status s = view(L, A, K, N, &v)) return s;
  // rank-natural source offsets: input order, positions ascending (chunk j before 2N-1-j)
  std::vector<int64_t> src_local(K, -1), src_lo(K, -1), src_hi(K, -1);
  int64_t s = 0;
  for (int32_t k = 0; k < K; ++k) {
    if (A[k] == j) {
      src_local[k] = s;
      s += L[k];
    } else if (A[k] == -1) {
      const int32_t c_lo = std::min(j, 2 * N - 1 - j), c_hi = std::max(j, 2 * N - 1 - j);
      Chunk x = chunk_of(L[k], c_lo, N), y = chunk_of(L[k], c_hi, N);
      src_lo[k] = s;
      s += x.b - x.a;
      src_hi[k] = s;
      s += y.b - y.a;
    }
  }
  int32_t seg = 0;
  int64_t row = 0;
  cu_seqlens_q[0] = 0;
  auto emit = [&](int32_t k, int32_t c, int64_t qpos, int64_t qlen, int64_t kstart, int64_t src0) {
    q_pos[seg] = (int32_t)qpos;
    k_len[seg] = (int32_t)(qpos + qlen);
    k_start[seg] = (int32_t)kstart;
    seg_seq[seg] = k;
    seg_chunk[seg] = c;
    for (int64_t r = 0; r < qlen; ++r) src_row[row + r] = (int32_t)(src0 + r);
    row += qlen;
    cu_seqlens_q[++seg] = (int32_t)row;
  };
  for (int32_t k : v.dist) {                       // R21: distributed prefix, chunk j then 2N-1-j
    for (int32_t c : {j, 2 * N - 1 - j}) {
      Chunk x = chunk_of(L[k], c, N);
      const int64_t src0 = (c == std::min(j, 2 * N - 1 - j)) ? src_lo[k] : src_hi[k];
      emit(k, c, x.a, x.b - x.a, v.nat_base[k], src0);
    }
  }
  for (int32_t k : v.order)                        // then locals on j in plan order
    if (A[k] == j) emit(k, -1, 0, L[k], row, src_local[k]);
  return SKR_OK;
}

SKR_EXPORT skr_status skr_pack_chunks(const int64_t* L, const int32_t* A, int32_t K, int32_t N,
                                      int32_t* table) {
  SKR_REQUIRE(N >= 1 && table, "skr_pack_chunks: bad arguments");
  MbView v;
  if (skr_status s = view(L, A, K, N, &v)) return s;
  int64_t P = 0;
  for (int32_t r = 0; r < N; ++r) P = std::max(P, dist_rows_of(L, v, N, r));
  // gathered_row = owner * P + offset < N * P must fit the int32 table (skr_pack_bounds checks the
  // same bound, but a C caller need not have called it first)
  if (P * N > INT32_MAX) return skr::fail(SKR_E_OVERFLOW, "skr_pack_chunks: N * P > 2^31 rows");
  // offset of each (seq, chunk) inside its owner's distributed prefix
  std::vector<int64_t> off_in_owner(N, 0);
  std::vector<int64_t> goff(2 * N * v.dist.size());
  for (size_t q = 0; q < v.dist.size(); ++q) {
    const int32_t k = v.dist[q];
    for (int32_t r = 0; r < N; ++r) {
      for (int32_t c : {r, 2 * N - 1 - r}) {
        Chunk x = chunk_of(L[k], c, N);
        goff[q * 2 * N + c] = off_in_owner[r];
        off_in_owner[r] += x.b - x.a;
      }
    }
  }
  int32_t* t = table;
  for (size_t q = 0; q < v.dist.size(); ++q) {
    const int32_t k = v.dist[q];
    for (int32_t c = 0; c < 2 * N; ++c) {
      Chunk x = chunk_of(L[k], c, N);
      const int32_t o = owner_of(c, N);
      t[0] = k;
      t[1] = c;
      t[2] = o;
      t[3] = (int32_t)(o * P + goff[q * 2 * N + c]);
      t[4] = (int32_t)(v.nat_base[k] + x.a);
      t[5] = (int32_t)(x.b - x.a);
      t += 6;
    }
  }
  return SKR_OK;
}

// Ring CP (row f4's alternative exchange): ring step `step` on rank j computes its own
// distributed query chunks against the K / V prefix of rank s = (j - step) mod N, which has travelled
// `step` hops along the ring. One segment per own query chunk (prefix order, so cu_seqlens_q tiles the
// rank's distributed prefix rows), against ONE key chunk of the visiting pair: cls 0 -> chunk s,
// cls 1 -> chunk 2N-1-s. Zigzag chunks are disjoint position ranges, so a key chunk before the query
// chunk is visible whole (q_pos = its length: every key precedes every query), the same chunk is the
// plain causal diagonal (q_pos = 0, only at step 0), a later chunk is invisible (k_len = 0: the
// attention calls write O = 0, LSE = -inf there). Over the N steps and both classes every key chunk
// c' <= c of a query chunk c is visited exactly once (see tests/test_host_planner.py).
SKR_EXPORT skr_status skr_ring_segs(const int64_t* L, const int32_t* A, int32_t K, int32_t N, int32_t j,
                                    int32_t step, int32_t cls, int32_t* cu_seqlens_q, int32_t* q_pos,
                                    int32_t* k_start, int32_t* k_len, int32_t cap, int32_t* n_seg) {
  SKR_REQUIRE(N >= 1 && j >= 0 && j < N && step >= 0 && step < N && (cls == 0 || cls == 1) && n_seg,
              "skr_ring_segs: bad rank / step / class");
  MbView v;
  if (skr_status st = view(L, A, K, N, &v)) return st;
  *n_seg = (int32_t)(2 * v.dist.size());
  if (*n_seg > cap) return fail(SKR_E_CAPACITY, "skr_ring_segs: need %d segments", *n_seg);
  SKR_REQUIRE(cu_seqlens_q && q_pos && k_start && k_len, "skr_ring_segs: null output");
  const int32_t s = ((j - step) % N + N) % N;
  const int32_t ck = cls == 0 ? s : 2 * N - 1 - s;
  int64_t qrow = 0, krow = 0;   // row in rank j's prefix / in the visiting (rank s's) prefix
  int32_t seg = 0;
  cu_seqlens_q[0] = 0;
  for (int32_t k : v.dist) {
    // key chunk ck's rows inside rank s's prefix (chunk s first, then 2N-1-s)
    const Chunk ks = chunk_of(L[k], s, N), kx = chunk_of(L[k], ck, N);
    const int64_t koff = krow + (ck == s ? 0 : ks.b - ks.a);
    const int64_t lk = kx.b - kx.a;
    for (int32_t c : {j, 2 * N - 1 - j}) {
      const Chunk q = chunk_of(L[k], c, N);
      const int64_t lq = q.b - q.a;
      if (lk == 0 || ck > c) {             // invisible
        q_pos[seg] = 0, k_start[seg] = 0, k_len[seg] = 0;
      } else if (ck < c) {                 // every key before every query
        q_pos[seg] = (int32_t)lk, k_start[seg] = (int32_t)koff, k_len[seg] = (int32_t)lk;
      } else {                             // the causal diagonal of the rank's own chunk
        q_pos[seg] = 0, k_start[seg] = (int32_t)koff, k_len[seg] = (int32_t)lk;
      }
      qrow += lq;
      cu_seqlens_q[++seg] = (int32_t)qrow;
    }
    const Chunk k2 = chunk_of(L[k], 2 * N - 1 - s, N);
    krow += (ks.b - ks.a) + (k2.b - k2.a);
  }
  return SKR_OK;
}

namespace {

struct Tile {
  int32_t seg, tile;
  int64_t work;
};

skr_status emit_tiles(std::vector<Tile>& v, int32_t* tiles, int32_t cap, int32_t* n_tiles) {
  // LPT: heaviest first; ties by (segment, tile) for determinism
  std::sort(v.begin(), v.end(), [](const Tile& a, const Tile& b) {
    if (a.work != b.work) return a.work > b.work;
    if (a.seg != b.seg) return a.seg < b.seg;
    return a.tile < b.tile;
  });
  *n_tiles = (int32_t)v.size();
  if ((int64_t)v.size() > cap) return skr::fail(SKR_E_CAPACITY, "tiles: need %zu entries", v.size());
  for (size_t i = 0; i < v.size(); ++i) tiles[2 * i] = v[i].seg, tiles[2 * i + 1] = v[i].tile;
  return SKR_OK;
}

}  // namespace

SKR_EXPORT skr_status skr_tiles_fwd(const int32_t* cu, const int32_t* q_pos, int32_t n_seg, int32_t bm,
                                    int32_t* tiles, int32_t cap, int32_t* n_tiles) {
  SKR_REQUIRE(n_tiles && bm > 0 && n_seg >= 0 && (n_seg == 0 || (cu && q_pos)) && (cap == 0 || tiles),
              "skr_tiles_fwd: bad arguments");
  std::vector<Tile> v;
  for (int32_t s = 0; s < n_seg; ++s) {
    const int64_t ql = cu[s + 1] - cu[s];
    SKR_REQUIRE(ql >= 0, "skr_tiles_fwd: cu_seqlens not monotone at %d", s);
    for (int64_t t = 0; t * bm < ql; ++t) {
      const int64_t last_key = q_pos[s] + std::min<int64_t>(ql, (t + 1) * bm);   // keys visible to the tile
      v.push_back({s, (int32_t)t, last_key});
    }
  }
  return emit_tiles(v, tiles, cap, n_tiles);
}

SKR_EXPORT skr_status skr_tiles_bwd(const int32_t* cu, const int32_t* q_pos, const int32_t* k_len, int32_t n_seg,
                                    int32_t bn, int32_t band_rows, int32_t* tiles, int32_t cap, int32_t* n_tiles) {
  SKR_REQUIRE(n_tiles && bn > 0 && n_seg >= 0 && (n_seg == 0 || (cu && q_pos && k_len)) && (cap == 0 || tiles),
              "skr_tiles_bwd: bad arguments");
  SKR_REQUIRE(band_rows >= 0 && band_rows % 128 == 0, "skr_tiles_bwd: band_rows %d must be a multiple of 128",
              band_rows);
  // Segments longer than band_rows are split into query bands [b * band_rows, (b + 1) * band_rows):
  // one work item per (key tile, band), ordered segment by segment, band by band, key tiles
  // ascending, so the CTAs in flight share one band's Q / dO / dQ rows (L2-resident) instead of each
  // streaming its key tile's whole query range. The rest: one item per key tile, LPT-ordered, after
  // the banded items (they also form the tail of the launch).
  struct Item {
    int32_t seg, tile, q_lo, q_hi;
    int64_t work;
  };
  std::vector<Item> banded, whole;
  for (int32_t s = 0; s < n_seg; ++s) {
    const int64_t ql = cu[s + 1] - cu[s];
    SKR_REQUIRE(ql >= 0, "skr_tiles_bwd: cu_seqlens not monotone at %d", s);
    if (ql <= 0) continue;
    const bool split = band_rows > 0 && ql > band_rows;
    const int64_t nb = split ? (ql + band_rows - 1) / band_rows : 1;
    for (int64_t b = 0; b < nb; ++b) {
      for (int64_t t = 0; t * bn < k_len[s]; ++t) {
        // queries (segment-relative) that see this key tile: [first_q, ql)
        const int64_t first_q = std::max<int64_t>(q_pos[s], t * bn) - q_pos[s];
        const int64_t lo = split ? b * band_rows : 0, hi = split ? std::min<int64_t>(ql, (b + 1) * band_rows) : ql;
        if (std::max(lo, first_q) >= hi) continue;
        (split ? banded : whole).push_back({s, (int32_t)t, (int32_t)lo, (int32_t)hi, hi - std::max(lo, first_q)});
      }
    }
  }
  // LPT for the whole-range items: heaviest first; ties by (segment, tile) for determinism
  std::sort(whole.begin(), whole.end(), [](const Item& a, const Item& b) {
    if (a.work != b.work) return a.work > b.work;
    if (a.seg != b.seg) return a.seg < b.seg;
    return a.tile < b.tile;
  });
  *n_tiles = (int32_t)(banded.size() + whole.size());
  if ((int64_t)*n_tiles > cap) return skr::fail(SKR_E_CAPACITY, "tiles: need %d entries", *n_tiles);
  int32_t* o = tiles;
  for (const auto* v : {&banded, &whole})
    for (const Item& x : *v) o[0] = x.seg, o[1] = x.tile, o[2] = x.q_lo, o[3] = x.q_hi, o += 4;
  return SKR_OK;
}

SKR_EXPORT skr_status skr_pack_owner_rows(const int32_t* table, int32_t n_chunks, int32_t natural_rows,
                                          int32_t* row_map) {
  SKR_REQUIRE(n_chunks >= 0 && natural_rows >= 0 && (n_chunks == 0 || table) && (natural_rows == 0 || row_map),
              "skr_pack_owner_rows: bad arguments");
  for (int32_t i = 0; i < natural_rows; ++i) row_map[i] = -1;
  for (int32_t c = 0; c < n_chunks; ++c) {
    const int32_t* t = table + 6 * c;
    const int64_t g = t[3], n = t[4], len = t[5];
    SKR_REQUIRE(len >= 0 && n >= 0 && n + len <= natural_rows && g >= 0 && g + len <= INT32_MAX,
                "skr_pack_owner_rows: chunk %d outside the natural rows", c);
    for (int64_t r = 0; r < len; ++r) row_map[n + r] = (int32_t)(g + r);
  }
  for (int32_t i = 0; i < natural_rows; ++i)
    SKR_REQUIRE(row_map[i] >= 0, "skr_pack_owner_rows: natural row %d has no chunk", i);
  return SKR_OK;
}
