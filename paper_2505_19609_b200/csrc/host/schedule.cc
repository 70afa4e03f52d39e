// a2/a3: Skrull's heuristics -- DACP (Alg. 1 + Alg. 3), GDS (Alg. 2,
// P:288-309) with its LPT binpack, and the Eq. 1-7 evaluator.
//
// Exact integer arithmetic (reading R4): the RemainBucket and Loads ledgers are kept scaled by N,
//   RB' = N*RB  (local: -N*S on one rank; distributed: -S on every rank)
//   L'  = N*L   (local: +N*F(S) on one rank; distributed: +F(S) on every rank)
// so S/N and FLOPs(S)/N (R5) never round and plans are bit-exact against any exact implementation.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../common.h"

namespace skr {
bool flops128(int64_t S, const skr_model& m, __int128* out);
}

namespace {

using i128 = __int128;
constexpr int32_t kUnassigned = INT32_MIN;

struct DacpOut {
  skr_status st = SKR_OK;
  int32_t n_rollbacks = 0;
  int32_t fail_pos = -1;
};

skr_status check_model(const skr_model* m) {
  if (!m || m->hidden < 1 || m->kv_hidden < 1 || m->pack_batch < 1)
    return skr::fail(SKR_E_ARG, "model fields must be >= 1");
  return SKR_OK;
}

// Alg. 1 on lens (input order); writes assign (input order).
DacpOut dacp_core(const int64_t* lens, int32_t K, int32_t N, int64_t C, bool rollback, const skr_model& m,
                  int32_t* assign) {
  DacpOut out;
  std::vector<int32_t> order(K);
  std::iota(order.begin(), order.end(), 0);
  // line 1 "Sort(SeqLens, ascending=True)", ties by input index (R1)
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return lens[a] != lens[b] ? lens[a] < lens[b] : a < b;
  });
  std::vector<int64_t> S(K);
  std::vector<i128> F(K);
  for (int32_t p = 0; p < K; ++p) {
    S[p] = lens[order[p]];
    skr::flops128(S[p], m, &F[p]);
  }
  // lines 2-3: RB[i] <- C, L[i] <- 0   (scaled by N, R4)
  std::vector<i128> RB(N, (i128)N * C), L(N, 0);
  std::vector<int32_t> ret(K, kUnassigned);                       // R9

  auto update_local = [&](int32_t p, int32_t r) {                 // Alg. 3 UpdateLocal
    RB[r] -= (i128)N * S[p];
    L[r] += (i128)N * F[p];
  };
  auto update_all = [&](int32_t p) {                              // Alg. 3 UpdateAll
    for (int32_t j = 0; j < N; ++j) {
      RB[j] -= S[p];                                              //   RB -= S/N  (scaled)
      L[j] += F[p];                                               //   L  += FLOPs(S)/N (R5, scaled)
    }
  };
  auto argmin = [&](const std::vector<i128>& a) {                 // lowest rank on ties (R2)
    int32_t t = 0;
    for (int32_t j = 1; j < N; ++j)
      if (a[j] < a[t]) t = j;
    return t;
  };
  auto argmax = [&](const std::vector<i128>& a) {
    int32_t t = 0;
    for (int32_t j = 1; j < N; ++j)
      if (a[j] > a[t]) t = j;
    return t;
  };

  int32_t i = 0;
  while (i < K) {                                                 // line 4
    int32_t t = argmin(L);                                        // line 5
    if (RB[t] >= (i128)N * S[i]) {                                // line 6: RB[t] >= S[i] (R3)
      ret[i] = t, update_local(i, t), ++i;
      continue;
    }
    t = argmax(RB);                                               // line 10
    if (RB[t] >= (i128)N * S[i]) {                                // line 11
      ret[i] = t, update_local(i, t), ++i;
      continue;
    }
    t = argmin(RB);                                               // line 14
    if (RB[t] >= (i128)S[i]) {                                    // line 15: RB[t] >= S[i]/N
      ret[i] = -1, update_all(i), ++i;                            // line 16: distribute
      continue;
    }
    // line 18: Assert RollBack(t, RB, L); Alg. 3 RollBack with the R6 erratum fix
    if (!rollback) {
      out.st = SKR_E_SCHEDULE, out.fail_pos = i;
      return out;
    }
    int32_t v = -1;
    for (int32_t q = 0; q < K; ++q)
      if (ret[q] == t) {                                          // first (shortest) local on t (R7)
        v = q;
        break;
      }
    if (v < 0) {
      out.st = SKR_E_SCHEDULE, out.fail_pos = i;
      return out;
    }
    ret[v] = -1;
    RB[t] += (i128)N * S[v];                                      // give the whole sequence back,
    L[t] -= (i128)N * F[v];
    update_all(v);                                                // then charge S/N to every rank
    ++out.n_rollbacks;                                            // lines 19-20: retry i (R8)
  }
  for (int32_t p = 0; p < K; ++p) assign[order[p]] = ret[p];
  return out;
}

}  // namespace

using skr::fail;

SKR_EXPORT skr_status skr_dacp(const int64_t* lens, int32_t K, const skr_cluster* cl, const skr_model* m,
                               int32_t* assign, int32_t* n_rollbacks, int32_t* fail_idx) {
  SKR_REQUIRE(cl && K >= 0 && (K == 0 || (lens && assign)), "skr_dacp: bad arguments");
  SKR_REQUIRE(cl->cp >= 1 && cl->bucket_tokens >= 0, "skr_dacp: cp must be >= 1, bucket >= 0");
  if (skr_status s = check_model(m)) return s;
  for (int32_t k = 0; k < K; ++k) SKR_REQUIRE(lens[k] >= 0, "skr_dacp: negative length at %d", k);
  DacpOut o = dacp_core(lens, K, cl->cp, cl->bucket_tokens, cl->rollback != 0, *m, assign);
  if (n_rollbacks) *n_rollbacks = o.n_rollbacks;
  if (fail_idx) *fail_idx = o.fail_pos;
  if (o.st) return fail(o.st, "DACP: sequence at sorted position %d cannot be placed (%s)", o.fail_pos,
                        cl->rollback ? "roll-back impossible" : "roll-back disabled");
  return SKR_OK;
}

SKR_EXPORT skr_status skr_eval_tdacp(const int64_t* lens, const int32_t* assign, int32_t K, const skr_cluster* cl,
                                     const skr_model* m, const skr_cost* cost, double* per_rank_time,
                                     double* comm_time, double* dist_time, double* tdacp, int32_t* feasible) {
  SKR_REQUIRE(cl && cost && K >= 0 && (K == 0 || (lens && assign)), "skr_eval_tdacp: bad arguments");
  if (skr_status s = check_model(m)) return s;
  const int32_t N = cl->cp;
  SKR_REQUIRE(N >= 1, "skr_eval_tdacp: cp must be >= 1");
  std::vector<i128> local(N, 0);
  std::vector<i128> used(N, 0);        // N * tokens on each rank (Eq. 7, scaled)
  i128 dist = 0, dist_tokens = 0;
  for (int32_t k = 0; k < K; ++k) {
    SKR_REQUIRE(assign[k] == -1 || (assign[k] >= 0 && assign[k] < N), "skr_eval_tdacp: bad assign[%d]", k);
    i128 f;
    skr::flops128(lens[k], *m, &f);
    if (assign[k] == -1) {
      dist += f;                                               // Eq. 4 numerator
      dist_tokens += lens[k];                                  // Eq. 5 argument
      for (int32_t j = 0; j < N; ++j) used[j] += lens[k];
    } else {
      local[assign[k]] += f;                                   // Eq. 3
      used[assign[k]] += (i128)N * lens[k];
    }
  }
  const double V = (double)(dist_tokens * m->pack_batch * m->kv_hidden) * cost->bytes_per_elem;   // Eq. 14
  const double tc = skr_t_comm(V, &cost->comm);                                                   // Eq. 15
  const double td = skr_t_comp((double)dist / N, &cost->comp) * cost->dist_penalty;               // Eq. 4, 13
  double best = 0;
  for (int32_t j = 0; j < N; ++j) {
    const double t = std::max(tc, skr_t_comp((double)local[j], &cost->comp)) + td;                // Eq. 2
    if (per_rank_time) per_rank_time[j] = t;
    best = std::max(best, t);                                                                     // Eq. 1
  }
  bool ok = true;
  for (int32_t j = 0; j < N; ++j) ok = ok && used[j] <= (i128)N * cl->bucket_tokens;            // Eq. 7
  if (comm_time) *comm_time = tc;
  if (dist_time) *dist_time = td;
  if (tdacp) *tdacp = K ? best : 0.0;
  if (feasible) *feasible = ok ? 1 : 0;
  return SKR_OK;
}

SKR_EXPORT skr_status skr_lpt(const int64_t* lens, int32_t K, int32_t bins, const skr_model* m,
                              int32_t* bin_of_seq) {
  SKR_REQUIRE(K >= 0 && bins >= 1 && (K == 0 || (lens && bin_of_seq)), "skr_lpt: bad arguments");
  if (skr_status s = check_model(m)) return s;
  std::vector<i128> F(K);
  for (int32_t k = 0; k < K; ++k) skr::flops128(lens[k], *m, &F[k]);
  std::vector<int32_t> idx(K);
  std::iota(idx.begin(), idx.end(), 0);
  // R16: FLOPs descending, ties by index; each to the bin with the smallest total (ties: lowest bin)
  std::sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return F[a] != F[b] ? F[a] > F[b] : a < b; });
  std::vector<i128> tot(bins, 0);
  for (int32_t k : idx) {
    int32_t best = 0;
    for (int32_t b = 1; b < bins; ++b)
      if (tot[b] < tot[best]) best = b;
    bin_of_seq[k] = best;
    tot[best] += F[k];
  }
  return SKR_OK;
}

namespace {

// Alg. 2 lines 2-8 for one subset (global indices); on success mb_of_seq[k] set for k in subset.
skr_status gds_core(const int64_t* lens, const std::vector<int32_t>& subset_in, const skr_cluster& cl,
                    const skr_model& m, int32_t* mb_of_seq, int32_t* n_mb) {
  std::vector<int32_t> sub = subset_in;
  std::sort(sub.begin(), sub.end(), [&](int32_t a, int32_t b) {   // line 3 (R18)
    return lens[a] != lens[b] ? lens[a] < lens[b] : a < b;
  });
  const i128 cap = (i128)cl.bucket_tokens * cl.cp;                 // C x N (Eq. 10)
  i128 total = 0;
  for (int32_t k : sub) total += lens[k];
  const int64_t n = (int64_t)sub.size();
  int64_t init = cap > 0 ? (int64_t)((total + cap - 1) / cap) : (total > 0 ? n + 2 : 1);
  if (init < 1) init = 1;                                          // line 2 (R11)
  std::vector<int64_t> mb_lens;
  std::vector<int32_t> scratch;
  for (; init <= n + 1; ++init) {                                  // line 4 (R15), line 5 (R14)
    bool ok = true;
    for (int64_t j = 0; j < init && ok; ++j) {                     // line 6 (R12)
      mb_lens.clear();
      i128 s = 0;
      for (int64_t q = j; q < n; q += init) mb_lens.push_back(lens[sub[q]]), s += lens[sub[q]];  // line 7
      if (s > cap) {                                               // line 8 (R13)
        ok = false;
        break;
      }
      scratch.assign(mb_lens.size(), 0);
      DacpOut o = dacp_core(mb_lens.data(), (int32_t)mb_lens.size(), cl.cp, cl.bucket_tokens, cl.rollback != 0, m,
                            scratch.data());
      if (o.st) ok = false;
    }
    if (ok) {
      for (int64_t q = 0; q < n; ++q) mb_of_seq[sub[q]] = (int32_t)(q % init);
      *n_mb = (int32_t)init;
      return SKR_OK;
    }
  }
  return skr::fail(SKR_E_GDS, "GDS: no feasible micro-batching up to init = %lld", (long long)(n + 1));
}

}  // namespace

SKR_EXPORT skr_status skr_gds(const int64_t* lens, int32_t K, const skr_cluster* cl, const skr_model* m,
                              int32_t dp_rank, int32_t* mb_of_seq, int32_t* n_mb) {
  SKR_REQUIRE(cl && n_mb && K >= 0 && (K == 0 || (lens && mb_of_seq)), "skr_gds: bad arguments");
  SKR_REQUIRE(cl->dp >= 1 && dp_rank >= 0 && dp_rank < cl->dp && cl->cp >= 1, "skr_gds: bad dp/cp");
  if (skr_status s = check_model(m)) return s;
  std::vector<int32_t> bin(K);
  if (skr_status s = skr_lpt(lens, K, cl->dp, m, bin.data())) return s;
  std::vector<int32_t> sub;
  for (int32_t k = 0; k < K; ++k) {
    mb_of_seq[k] = -1;
    if (bin[k] == dp_rank) sub.push_back(k);
  }
  *n_mb = 0;
  if (sub.empty()) return SKR_OK;
  return gds_core(lens, sub, *cl, *m, mb_of_seq, n_mb);
}

SKR_EXPORT skr_status skr_plan(const int64_t* lens, int32_t K, const skr_cluster* cl, const skr_model* m,
                               int32_t* dp_of_seq, int32_t* mb_of_seq, int32_t* assign, int32_t* n_mb_per_dp,
                               int32_t* n_rollbacks) {
  SKR_REQUIRE(cl && n_mb_per_dp && K >= 0 && (K == 0 || (lens && dp_of_seq && mb_of_seq && assign)),
              "skr_plan: bad arguments");
  SKR_REQUIRE(cl->dp >= 1 && cl->cp >= 1, "skr_plan: bad dp/cp");
  if (skr_status s = check_model(m)) return s;
  if (skr_status s = skr_lpt(lens, K, cl->dp, m, dp_of_seq)) return s;
  int32_t nrb = 0;
  std::vector<int64_t> mb_lens;
  std::vector<int32_t> mb_idx, mb_asg;
  for (int32_t i = 0; i < cl->dp; ++i) {
    std::vector<int32_t> sub;
    for (int32_t k = 0; k < K; ++k)
      if (dp_of_seq[k] == i) sub.push_back(k);
    n_mb_per_dp[i] = 0;
    if (sub.empty()) continue;
    if (skr_status s = gds_core(lens, sub, *cl, *m, mb_of_seq, &n_mb_per_dp[i])) return s;
    for (int32_t j = 0; j < n_mb_per_dp[i]; ++j) {                                    // DACP per mb
      mb_lens.clear(), mb_idx.clear();
      for (int32_t k : sub)        // stride-of-sorted order is ascending; DACP sorts anyway (R1)
        if (mb_of_seq[k] == j) mb_idx.push_back(k), mb_lens.push_back(lens[k]);
      mb_asg.assign(mb_idx.size(), 0);
      DacpOut o = dacp_core(mb_lens.data(), (int32_t)mb_lens.size(), cl->cp, cl->bucket_tokens,
                            cl->rollback != 0, *m, mb_asg.data());
      if (o.st) return fail(SKR_E_SCHEDULE, "skr_plan: DACP failed on dp %d micro-batch %d", i, j);
      nrb += o.n_rollbacks;
      for (size_t q = 0; q < mb_idx.size(); ++q) assign[mb_idx[q]] = mb_asg[q];
    }
  }
  if (n_rollbacks) *n_rollbacks = nrb;
  return SKR_OK;
}

// ---------------------------------------------------------------------------- baselines (row f1)
// Alg. 4 round-robin (reading R27: all K sequences in input order, shard by N), with the
// R6 roll-back on the RemainBucket ledger only (RR keeps no load array), and the DeepSpeed-like
// full-shard plan: FIFO micro-batches under C*N tokens, all distributed.
SKR_EXPORT skr_status skr_round_robin(const int64_t* lens, int32_t K, const skr_cluster* cl, int32_t* assign,
                                      int32_t* n_rollbacks, int32_t* fail_idx) {
  SKR_REQUIRE(cl && K >= 0 && (K == 0 || (lens && assign)) && cl->cp >= 1, "skr_round_robin: bad arguments");
  const int32_t N = cl->cp;
  std::vector<i128> RB(N, (i128)N * cl->bucket_tokens);   // scaled by N (R4)
  std::vector<int32_t> ret(K, kUnassigned);
  int32_t nrb = 0;
  int32_t i = 0;
  while (i < K) {
    SKR_REQUIRE(lens[i] >= 0, "skr_round_robin: negative length");
    int32_t t = 0;                                        // FindMaxBucketsIds (lowest on ties)
    for (int32_t j = 1; j < N; ++j)
      if (RB[j] > RB[t]) t = j;
    if (RB[t] >= (i128)N * lens[i]) {
      ret[i] = t, RB[t] -= (i128)N * lens[i], ++i;
      continue;
    }
    int32_t m = 0;                                        // FindMinBucketsIds
    for (int32_t j = 1; j < N; ++j)
      if (RB[j] < RB[m]) m = j;
    if (RB[m] >= (i128)lens[i]) {                          // C[j] >= S[i]/N
      ret[i] = -1;
      for (int32_t j = 0; j < N; ++j) RB[j] -= lens[i];
      ++i;
      continue;
    }
    int32_t v = -1;
    if (cl->rollback)
      for (int32_t q = 0; q < K; ++q)
        if (ret[q] == m) {
          v = q;
          break;
        }
    if (v < 0) {
      if (fail_idx) *fail_idx = i;
      if (n_rollbacks) *n_rollbacks = nrb;
      return fail(SKR_E_SCHEDULE, "round-robin: sequence %d cannot be placed (%s)", i,
                  cl->rollback ? "roll-back impossible" : "roll-back disabled");
    }
    ret[v] = -1;
    RB[m] += (i128)N * lens[v];
    for (int32_t j = 0; j < N; ++j) RB[j] -= lens[v];
    ++nrb;
  }
  for (int32_t k = 0; k < K; ++k) assign[k] = ret[k];
  if (n_rollbacks) *n_rollbacks = nrb;
  if (fail_idx) *fail_idx = -1;
  return SKR_OK;
}

SKR_EXPORT skr_status skr_full_shard(const int64_t* lens, int32_t K, const skr_cluster* cl, int32_t* mb_of_seq,
                                     int32_t* n_mb) {
  SKR_REQUIRE(cl && n_mb && K >= 0 && (K == 0 || (lens && mb_of_seq)) && cl->cp >= 1,
              "skr_full_shard: bad arguments");
  const i128 cap = (i128)cl->bucket_tokens * cl->cp;
  int32_t mb = 0;
  i128 tot = 0;
  bool open = false;
  for (int32_t k = 0; k < K; ++k) {
    if (lens[k] > (i128)cl->bucket_tokens * cl->cp)
      return fail(SKR_E_SCHEDULE, "full-shard: sequence %d (%lld tokens) exceeds C*N", k, (long long)lens[k]);
    if (open && tot + lens[k] > cap) ++mb, tot = 0;
    mb_of_seq[k] = mb;
    tot += lens[k];
    open = true;
  }
  *n_mb = open ? mb + 1 : 0;
  return SKR_OK;
}
