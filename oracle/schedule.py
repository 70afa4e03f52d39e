"""Oracle: Skrull's schedulers (§4.3.2, Alg. 1-3)
and the DACP / joint objectives (Eq. 1-11), in exact Fraction arithmetic.

Test infrastructure only (see oracle/__init__.py).

Readings applied (DESIGN.md ledger): R1 stable ascending sort, R2 lowest-rank
tie-break, R3 inclusive >=, R5 FLOPs(S,N) = FLOPs(S)/N, R6 RollBack erratum
fix, R7 shortest-local victim, R8 retry same sequence, R9 unassigned sentinel,
R11-R16 GDS/LPT details, R18 micro-batch order.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from fractions import Fraction

from .cost_model import Fit, Model, flops, t_comm, t_comp, volume

UNASSIGNED = None


class ScheduleError(Exception):
    """Alg. 1's Assert fails or roll-back disabled (Table 3 'OOM')."""

    def __init__(self, pos: int):
        super().__init__(f"DACP scheduling failed at sorted position {pos}")
        self.pos = pos


class GDSError(Exception):
    """No init <= |Subset|+1 gives all-feasible micro-batches (Alg. 2; R15)."""


@dataclass
class DacpResult:
    assign: list          # input order: -1 distributed, v in [0,N) local on CP rank v
    n_rollbacks: int
    RB: list              # final RemainBucket (Fractions, tokens)
    L: list               # final Loads (Fractions, FLOPs)


def dacp(lens, C: int, N: int, m: Model, rollback: bool = True) -> DacpResult:
    """Algorithm 1 with Algorithm 3's UpdateLocal / UpdateAll / RollBack."""
    K = len(lens)
    order = sorted(range(K), key=lambda k: (lens[k], k))        # line 1 "Sort ascending" (R1)
    S = [int(lens[k]) for k in order]
    RB = [Fraction(C) for _ in range(N)]                         # lines 2-3 RB[i] <- C
    L = [Fraction(0) for _ in range(N)]                          #           L[i] <- 0
    ret = [UNASSIGNED] * K                                       # R9
    n_rb = 0

    def update_local(idx, rank):                                 # Alg. 3 UpdateLocal
        RB[rank] -= S[idx]
        L[rank] += flops(S[idx], m)

    def update_all(idx):                                         # Alg. 3 UpdateAll
        for i in range(N):
            RB[i] -= Fraction(S[idx], N)
            L[i] += Fraction(flops(S[idx], m), N)                # FLOPs(S,N) = FLOPs(S)/N (R5)

    def roll_back(rank) -> bool:                                 # Alg. 3 RollBack
        for i in range(K):
            if ret[i] == rank:                                   # first local on `rank` (R7)
                ret[i] = -1
                # R6 erratum: restore the whole sequence to `rank`, then charge S/N
                # and FLOPs/N to every rank (an UpdateAll), so Eq. 7 accounting holds.
                RB[rank] += S[i]
                L[rank] -= flops(S[i], m)
                update_all(i)
                return True
        return False

    def argmin(a):                                               # lowest index on ties (R2)
        return min(range(N), key=lambda j: (a[j], j))

    def argmax(a):
        return min(range(N), key=lambda j: (-a[j], j))

    i = 0
    while i < K:                                                 # line 4 "for i = 0 to K-1"
        t = argmin(L)                                            # line 5
        if RB[t] >= S[i]:                                        # line 6 (R3)
            ret[i] = t
            update_local(i, t)
            i += 1
            continue
        t = argmax(RB)                                           # line 10
        if RB[t] >= S[i]:                                        # line 11
            ret[i] = t
            update_local(i, t)
            i += 1
            continue
        t = argmin(RB)                                           # line 14
        if RB[t] >= Fraction(S[i], N):                           # line 15
            ret[i] = -1
            update_all(i)
            i += 1
            continue
        if not rollback or not roll_back(t):                     # line 18 "Assert RollBack"
            raise ScheduleError(i)
        n_rb += 1                                                # lines 19-20: i <- i-1; continue (R8)
    assign = [0] * K
    for p, k in enumerate(order):
        assign[k] = ret[p]
    return DacpResult(assign, n_rb, RB, L)


# ---------------------------------------------------------------------------
# Eq. 1-7 evaluator
# ---------------------------------------------------------------------------

@dataclass
class TdacpBreakdown:
    per_rank_time: list
    comm_time: object
    dist_time: object
    local_time: list
    tdacp: object
    feasible: bool
    residual: list


def check_feasible(lens, assign, C, N):
    """Eq. 7: sum_k S_k P_kj + D_k S_k / N <= C for every rank j."""
    used = [Fraction(0)] * N
    for S, a in zip(lens, assign):
        if a == -1:
            for j in range(N):
                used[j] += Fraction(int(S), N)
        else:
            used[a] += int(S)
    resid = [Fraction(C) - u for u in used]
    return all(r >= 0 for r in resid), resid


def eval_tdacp(lens, assign, C, N, m: Model, comp: Fit, comm: Fit,
               bytes_per_elem: float = 1, dist_penalty=1):
    """Eq. 1-5. Time_j = max(T_comm(V), T_comp(Local_j)) + T_comp(Dist).

    Local_j = sum FLOPs of locals on j (Eq. 3); Dist = (1/N) sum FLOPs of distributed (Eq. 4);
    V = Volume(sum_k D_k S_k) (Eq. 5) in elements * bytes_per_elem (R25). `dist_penalty`
    multiplies T_comp(Dist): the per-shard kernel-efficiency penalty of the FIT_TEST preset
    (Fig. 1b) -- 1 means Eq. 2 exactly.
    """
    local = [0] * N
    dist = 0
    dist_tokens = 0
    for S, a in zip(lens, assign):
        if a == -1:
            dist += flops(int(S), m)
            dist_tokens += int(S)
        else:
            local[a] += flops(int(S), m)
    dist_f = Fraction(dist, N)
    V = volume(dist_tokens, m) * bytes_per_elem
    tc = t_comm(V, comm)
    td = t_comp(dist_f, comp) * dist_penalty
    tl = [t_comp(x, comp) for x in local]
    per = [max(tc, x) + td for x in tl]
    feas, resid = check_feasible(lens, assign, C, N)
    return TdacpBreakdown(per, tc, td, tl, max(per) if per else 0, feas, resid)


def overlap_gain(b: TdacpBreakdown):
    """Fig. 3(d) diagnostic: mean over ranks of (comm + local) - max(comm, local)."""
    N = len(b.local_time)
    return sum((b.comm_time + x) - max(b.comm_time, x) for x in b.local_time) / N


def optimal_dacp(lens, C, N, m: Model, comp: Fit, comm: Fit, bytes_per_elem=1,
                 dist_penalty=1, max_k: int = 8):
    """Exhaustive optimum of Eq. 1 subject to Eq. 6-7 over {-1, 0..N-1}^K.

    Ties -> lexicographically smallest assignment (itertools.product order with -1 first).
    Returns (assign, tdacp) or None when no assignment satisfies Eq. 7.
    """
    K = len(lens)
    if K > max_k:
        raise ValueError("K too large for exhaustive search")
    best = None
    for a in itertools.product([-1] + list(range(N)), repeat=K):
        feas, _ = check_feasible(lens, a, C, N)
        if not feas:
            continue
        t = eval_tdacp(lens, a, C, N, m, comp, comm, bytes_per_elem, dist_penalty).tdacp
        if best is None or t < best[1]:
            best = (list(a), t)
    return best


# ---------------------------------------------------------------------------
# GDS (Alg. 2) and the binpack of its line 1
# ---------------------------------------------------------------------------

def lpt(lens, bins: int, m: Model):
    """Alg. 2 line 1 'Binpack(ws, FLOPs(S[K]))' as greedy LPT (R16):
    indices by FLOPs descending (ties by index) to the bin with the smallest total (ties lowest)."""
    tot = [0] * bins
    out = [0] * len(lens)
    for k in sorted(range(len(lens)), key=lambda k: (-flops(int(lens[k]), m), k)):
        i = min(range(bins), key=lambda b: (tot[b], b))
        out[k] = i
        tot[i] += flops(int(lens[k]), m)
    return out


def gds(lens, subset, C, N, m: Model, rollback=True):
    """Alg. 2 lines 2-8 for one DP rank's `subset` (global indices).

    Returns a list of micro-batches (lists of global indices, ascending by length).
    R11 init0 = max(1, ceil(sum/(C*N))); R12 j in [0, init); R13 overload iff sum > C*N;
    R14 any failure aborts this init; R15 give up past len(subset)+1.
    """
    sub = sorted(subset, key=lambda k: (lens[k], k))            # line 3 (R18)
    total = sum(int(lens[k]) for k in sub)
    init = max(1, -(-total // (C * N)))                          # line 2 (R11)
    while init <= len(sub) + 1:                                  # line 4 (R15)
        mbs = [sub[j::init] for j in range(init)]                # lines 6-7 (R12)
        ok = True
        for mb in mbs:
            if sum(int(lens[k]) for k in mb) > C * N:            # line 8 (R13: Eq. 10 normative)
                ok = False
                break
            try:
                dacp([lens[k] for k in mb], C, N, m, rollback)
            except ScheduleError:
                ok = False
                break
        if ok:
            return mbs
        init += 1                                                # line 5 on the next pass (R14)
    raise GDSError("no feasible micro-batching")


@dataclass
class Plan:
    dp_of_seq: list
    mb_of_seq: list       # micro-batch index within its DP rank
    assign: list          # DACP result within its micro-batch
    n_mb: list            # per DP rank
    mbs: list             # mbs[i][j] = list of global indices (ascending by length)
    n_rollbacks: int


def plan(lens, C, N, ws, m: Model, rollback=True) -> Plan:
    """Full iteration plan: LPT bins, GDS per DP rank,
    DACP per micro-batch."""
    K = len(lens)
    dp = lpt(lens, ws, m)
    mb_of = [0] * K
    asg = [0] * K
    n_mb = []
    all_mbs = []
    nrb = 0
    for i in range(ws):
        sub = [k for k in range(K) if dp[k] == i]
        mbs = gds(lens, sub, C, N, m, rollback) if sub else []
        n_mb.append(len(mbs))
        all_mbs.append(mbs)
        for j, mb in enumerate(mbs):
            r = dacp([lens[k] for k in mb], C, N, m, rollback)
            nrb += r.n_rollbacks
            for k, a in zip(mb, r.assign):
                mb_of[k] = j
                asg[k] = a
    return Plan(dp, mb_of, asg, n_mb, all_mbs, nrb)


def eval_iteration(lens, p: Plan, C, N, m, comp, comm, bytes_per_elem=1, dist_penalty=1):
    """Eq. 8: max over DP ranks i of sum_j Time_ij, Time_ij = TDACP(mb_ij) (Eq. 11)."""
    per_dp = []
    for i, mbs in enumerate(p.mbs):
        s = 0
        for mb in mbs:
            s += eval_tdacp([lens[k] for k in mb], [p.assign[k] for k in mb], C, N, m,
                            comp, comm, bytes_per_elem, dist_penalty).tdacp
        per_dp.append(s)
    return max(per_dp) if per_dp else 0, per_dp


def optimal_joint_ws1(lens, C, N, m, comp, comm, bytes_per_elem=1, dist_penalty=1):
    """Joint GDS+DACP optimum (Eq. 8-11) for ws=1, K<=8: every set
    partition of the batch into micro-batches of <= C*N tokens (Eq. 10), each scored by
    its exhaustive DACP optimum; objective = sum over micro-batches (Eq. 8)."""
    K = len(lens)
    if K > 8:
        raise ValueError("K too large")
    cache = {}

    def best_mb(idx):
        key = tuple(sorted(idx))
        if key not in cache:
            ls = [lens[k] for k in key]
            if sum(ls) > C * N:
                cache[key] = None
            else:
                r = optimal_dacp(ls, C, N, m, comp, comm, bytes_per_elem, dist_penalty)
                cache[key] = None if r is None else r[1]
        return cache[key]

    best = None

    def rec(rest, acc):
        nonlocal best
        if not rest:
            if best is None or acc < best:
                best = acc
            return
        first, others = rest[0], rest[1:]
        for r in range(len(others) + 1):
            for comb in itertools.combinations(others, r):
                t = best_mb((first,) + comb)
                if t is None:
                    continue
                rec(tuple(x for x in others if x not in comb), acc + t)

    rec(tuple(range(K)), 0)
    return best


# ---------------------------------------------------------------------------
# Baselines (NEXT-1): Alg. 4 round-robin and the full-shard DeepSpeed-like plan
# ---------------------------------------------------------------------------

def round_robin(lens, C, N, rollback=True):
    """Alg. 4, input order (no sort), shard by N (R27); roll-back as R6 on RB only."""
    K = len(lens)
    RB = [Fraction(C)] * N
    ret = [UNASSIGNED] * K
    i = 0
    while i < K:
        S = int(lens[i])
        t = min(range(N), key=lambda j: (-RB[j], j))             # FindMaxBucketsIds
        if RB[t] >= S:
            ret[i] = t
            RB[t] -= S
            i += 1
            continue
        j = min(range(N), key=lambda q: (RB[q], q))              # FindMinBucketsIds
        if RB[j] >= Fraction(S, N):
            ret[i] = -1
            for q in range(N):
                RB[q] -= Fraction(S, N)
            i += 1
            continue
        if not rollback:
            raise ScheduleError(i)
        victim = next((q for q in range(K) if ret[q] == j), None)
        if victim is None:
            raise ScheduleError(i)
        ret[victim] = -1
        RB[j] += int(lens[victim])
        for q in range(N):
            RB[q] -= Fraction(int(lens[victim]), N)
    return ret


def full_shard(lens, C, N):
    """S:398-406 model of the paper's DeepSpeed baseline: FIFO micro-batches
    under the C*N token budget (Eq. 10), every sequence distributed."""
    mbs, cur, tot = [], [], 0
    for k, S in enumerate(lens):
        if Fraction(int(S), N) > C:
            raise ScheduleError(k)
        if cur and tot + int(S) > C * N:
            mbs.append(cur)
            cur, tot = [], 0
        cur.append(k)
        tot += int(S)
    if cur:
        mbs.append(cur)
    return mbs
