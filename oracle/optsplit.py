"""Oracle: per-node time model, OptPerf and the local-batch split r_opt.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Model (§3.2):
    a_i = q_i b_i + s_i,  P_i = k_i b_i + m_i                    (Eq. 3)
    syncStart_i = a_i + gamma P_i                                 (Eq. 4)
    compute-bound iff (1 - gamma) P_i >= T_o
    compute-bound node time  t_compute^i + T_u = a_i + P_i + T_u  (Eq. 5)
    comm-bound node time     syncStart_i + T_comm                 (Eq. 6)
    cluster time T = max{ max_i (t_compute^i + T_u), max_i (syncStart_i + T_comm) }   (Eq. 7)
and OptPerf = min over splits with sum_i b_i = B (§3.1).

Per node, Eq. 7 is f_i(b) = a_i + max(P_i, gamma P_i + T_o) + T_u, which equals Eq. 5 when the node
is compute-bound and Eq. 6 otherwise.  The *frozen evaluation contract* (reading O-5)
fixes the floating-point order so integer decisions are reproducible bit-for-bit:
    P = k*b + m;  A = q*b + s;  X = gamma*P + t_o;  f = (A + max(P, X)) + t_u
(binary64, left to right, no FMA -- Python floats never contract).

Solutions:
* ``real_split``   -- the relaxation's optimum: the smallest T with sum_i clamp(f_i^{-1}(T)) >= B,
  found by plain bisection.  At it all unclamped nodes finish together: compute-bound nodes share
  t_compute and comm-bound nodes share syncStart with t_compute = syncStart + T_o (the KKT
  conditions of App. A; §3.3).
* ``int_split_greedy`` -- the integer optimum of Eq. 7: starting at lo, hand out the B - sum(lo)
  samples one at a time to argmin_i (f_i(b_i + 1), i).  Integer batches are required.
* ``int_split_brute`` -- exhaustive enumeration (tiny n, B) with the canonical tie-break.
* ``algorithm1``   -- Alg. 1 literally, as a cross-check of ``real_split`` (its node-fixing
  rule is unsound, so it can fail).
* ``round_paper``  -- the paper's own integer rule: round the real split, implemented
  as largest-remainder with ties to the lower index.
* ``warmup_split`` -- Eq. 8.
"""
from __future__ import annotations

import itertools
import math


# ----------------------------------------------------------------------------- Eq. 3-7 pieces
def compute_time(node, b: float) -> float:
    """Eq. 3: t_compute = a + P = (q b + s) + (k b + m)."""
    q, s, k, m = node
    return (q * b + s) + (k * b + m)


def sync_start(node, comm, b: float) -> float:
    """Eq. 4: syncStart = a + gamma P."""
    q, s, k, m = node
    gamma = comm[0]
    return (q * b + s) + gamma * (k * b + m)


def is_compute_bound(node, comm, b: float) -> bool:
    """compute-bound iff (1 - gamma) P >= T_o (ties count as compute, the paper's ">=")."""
    q, s, k, m = node
    gamma, t_o, _ = comm
    return (1.0 - gamma) * (k * b + m) >= t_o


def node_time(node, comm, b: float) -> float:
    """Per-node term of Eq. 7 under the frozen evaluation contract."""
    q, s, k, m = node
    gamma, t_o, t_u = comm
    P = k * b + m
    A = q * b + s
    X = gamma * P + t_o
    return (A + max(P, X)) + t_u


def cluster_time(nodes, comm, b) -> float:
    """Eq. 7 as max_i f_i(b_i)."""
    return max(node_time(nodes[i], comm, float(b[i])) for i in range(len(nodes)))


def eq7_time(nodes, comm, b) -> float:
    """Eq. 7 written exactly as printed, for pinning ``cluster_time``."""
    gamma, t_o, t_u = comm
    t_comm = t_o + t_u
    first = max(compute_time(nodes[i], float(b[i])) + t_u for i in range(len(nodes)))
    second = max(sync_start(nodes[i], comm, float(b[i])) + t_comm for i in range(len(nodes)))
    return max(first, second)


# ----------------------------------------------------------------------------- validation
def _bounds(n, B, lo, cap):
    lo = [1] * n if lo is None else [int(x) for x in lo]
    cap = [int(B)] * n if cap is None else [int(x) for x in cap]
    if sum(lo) > B or sum(cap) < B or any(l > c for l, c in zip(lo, cap)):
        raise ValueError("infeasible bounds")
    return lo, cap


def _check_models(nodes, comm):
    gamma, t_o, t_u = comm
    if not (0.0 <= gamma < 1.0) or t_o < 0.0 or t_u < 0.0:
        raise ValueError("domain: need 0 <= gamma < 1, t_o >= 0, t_u >= 0")
    for q, s, k, m in nodes:
        if min(q, s, k, m) < 0.0:
            raise ValueError("domain: negative coefficient")
        if q + k == 0.0 or q + gamma * k == 0.0:
            # f must grow with b on both branches (Eq. 5 slope q+k, Eq. 6 slope q+gamma k),
            # otherwise the relaxation has a flat stretch and r_opt is not unique (Q18)
            raise ZeroDivisionError("singular: node time independent of b")


# ----------------------------------------------------------------------------- real r_opt
def node_inverse(node, comm, T: float) -> float:
    """Largest real b with f(b) <= T.  f = max(line1, line2) with
    line1 = (q + k) b + (s + m + t_u)            (compute-bound branch, Eq. 5)
    line2 = (q + gamma k) b + (s + gamma m + t_o + t_u)   (comm-bound branch, Eq. 6)
    so f^{-1}(T) = min(line1^{-1}(T), line2^{-1}(T))."""
    q, s, k, m = node
    gamma, t_o, t_u = comm
    inv1 = (T - (s + m + t_u)) / (q + k)
    slope2 = q + gamma * k
    c2 = s + gamma * m + t_o + t_u
    if slope2 > 0.0:
        inv2 = (T - c2) / slope2
    else:
        inv2 = math.inf if T >= c2 else -math.inf
    return min(inv1, inv2)


def real_split(nodes, comm, B: int, lo=None, cap=None):
    """Relaxed OptPerf split by bisection on T.  Returns (b_real, T_real, labels).

    T* = min{T : sum_i clamp(f_i^{-1}(T), lo_i, cap_i) >= B};  b_real_i = clamp(f_i^{-1}(T*));
    T_real = Eq. 7 at b_real;  labels[i] = 1 (compute-bound) or 0 (comm-bound).
    """
    _check_models(nodes, comm)
    n = len(nodes)
    lo, cap = _bounds(n, B, lo, cap)

    def h(T):
        tot = 0.0
        for i in range(n):
            tot += min(max(node_inverse(nodes[i], comm, T), float(lo[i])), float(cap[i]))
        return tot

    if sum(lo) == B:
        b = [float(x) for x in lo]
    else:
        t_lo = min(node_time(nodes[i], comm, float(lo[i])) for i in range(n)) - 1.0
        t_hi = max(node_time(nodes[i], comm, float(cap[i])) for i in range(n))
        while h(t_hi) < B:
            t_hi = 2.0 * t_hi + 1.0
        while True:
            mid = 0.5 * (t_lo + t_hi)
            if mid <= t_lo or mid >= t_hi:
                break
            if h(mid) >= B:
                t_hi = mid
            else:
                t_lo = mid
        b = [min(max(node_inverse(nodes[i], comm, t_hi), float(lo[i])), float(cap[i]))
             for i in range(n)]
    T = cluster_time(nodes, comm, b)
    labels = [1 if is_compute_bound(nodes[i], comm, b[i]) else 0 for i in range(n)]
    return b, T, labels


# ----------------------------------------------------------------------------- Algorithm 1, literally
def _solve_equal(lines, B: float):
    """Solve slope_i b_i + c_i = t for every i with sum_i b_i = B (unclamped):
    t = (B + sum_i c_i / slope_i) / sum_i (1 / slope_i),  b_i = (t - c_i) / slope_i."""
    num = float(B)
    den = 0.0
    for a, c in lines:
        num += c / a
        den += 1.0 / a
    t = num / den
    return t, [(t - c) / a for a, c in lines]


def breakpoint_time(node, comm) -> float:
    """T_i* = f_i(b_i^bp), b_i^bp = (T_o / (1 - gamma) - m_i) / k_i: the node's time where it turns
    compute-bound.  The ranking key of the mixed search (reading Q14)."""
    q, s, k, m = node
    gamma, t_o, _ = comm
    if k <= 0.0:
        return math.inf if (1.0 - gamma) * m < t_o else -math.inf
    return node_time(node, comm, (t_o / (1.0 - gamma) - m) / k)


def algorithm1(nodes, comm, B: float):
    """PAPER.md Algorithm 1, step by step, on the relaxation (real b, no bounds).

    Check 1: solve t_compute^0 = ... = t_compute^{n-1} with sum b = B; if every node is
      compute-bound ((1 - gamma) P_i >= T_o) return OptPerf = t_compute + T_u.
    Check 2: solve syncStart_0 = ... = syncStart_{n-1}; if every node is comm-bound
      return OptPerf = syncStart + T_comm.
    Mixed: a node with the same state in Check 1 and Check 2 keeps it; the
      other "outliers" are ranked by their breakpoint time (reading Q14: the undefined "fixed
      processing time"), nodes before the boundary C are computing-bottleneck, the rest
      communication-bottleneck; for each candidate boundary solve
      T_comb = t_compute' = syncStart' + T_o and test
      (forall syncStart_i <= syncStart') and (forall t_compute_i <= t_compute'); the
      boundary moves by bisection (reading Q16: a comm-labelled node that is really compute-bound
      moves it up, a compute-labelled node that is really comm-bound moves it down).
      OptPerf = T_comb + T_u.
    Returns {"b", "T", "case", "labels"} or None when no boundary gives a consistent state (the
    fixing rule of P:310 is unsound: the exact solver is ``real_split``)."""
    _check_models(nodes, comm)
    gamma, t_o, t_u = comm
    n = len(nodes)
    comp_line = [(q + k, s + m) for q, s, k, m in nodes]               # t_compute_i = a b + c
    sync_line = [(q + gamma * k, s + gamma * m) for q, s, k, m in nodes]  # syncStart_i = a b + c

    def state(i, b):
        return is_compute_bound(nodes[i], comm, b)

    # Check 1
    t1, b1 = _solve_equal(comp_line, B)
    lab1 = [state(i, b1[i]) for i in range(n)]
    if all(lab1):
        return {"b": b1, "T": t1 + t_u, "case": "compute", "labels": [1] * n}
    # Check 2
    s2, b2 = _solve_equal(sync_line, B)
    lab2 = [state(i, b2[i]) for i in range(n)]
    if not any(lab2):
        return {"b": b2, "T": s2 + t_o + t_u, "case": "comm", "labels": [0] * n}
    # mixed-bottleneck search
    fixed = {i: lab1[i] for i in range(n) if lab1[i] == lab2[i]}
    outliers = sorted((i for i in range(n) if lab1[i] != lab2[i]),
                      key=lambda i: (breakpoint_time(nodes[i], comm), i))
    beg, end = 0, len(outliers)
    while beg <= end:
        C = (beg + end) // 2
        is_comp = dict(fixed)
        for j, i in enumerate(outliers):
            is_comp[i] = j < C
        # T_comb = t_compute' = syncStart' + T_o: compute nodes a b + c = T_comb, comm nodes
        # a' b + c' + T_o = T_comb
        lines = [comp_line[i] if is_comp[i] else (sync_line[i][0], sync_line[i][1] + t_o)
                 for i in range(n)]
        t_comb, b = _solve_equal(lines, B)
        up = any((not is_comp[i]) and compute_time(nodes[i], b[i]) > t_comb for i in range(n))
        down = any(is_comp[i] and sync_start(nodes[i], comm, b[i]) > t_comb - t_o
                   for i in range(n))
        if not up and not down:
            return {"b": b, "T": t_comb + t_u, "case": "mixed",
                    "labels": [1 if is_comp[i] else 0 for i in range(n)]}
        if up and down:
            return None
        if up:
            beg = C + 1
        else:
            end = C - 1
    return None


# ----------------------------------------------------------------------------- integer splits
def int_split_greedy(nodes, comm, B: int, lo=None, cap=None):
    """Exact integer optimum of Eq. 7 with the canonical tie-break (lowest (f_i(b_i+1), i) first)."""
    _check_models(nodes, comm)
    n = len(nodes)
    lo, cap = _bounds(n, B, lo, cap)
    b = list(lo)
    for _ in range(B - sum(lo)):
        best = None
        for i in range(n):
            if b[i] < cap[i]:
                key = (node_time(nodes[i], comm, float(b[i] + 1)), i)
                if best is None or key < best:
                    best = key
        b[best[1]] += 1
    return b, cluster_time(nodes, comm, b)


def int_split_brute(nodes, comm, B: int, lo=None, cap=None):
    """Enumerate every integer split with lo <= b <= cap, sum = B.  Pick the one whose multiset of
    marginal keys {(f_i(j), i) : lo_i < j <= b_i}, sorted descending, is lexicographically
    smallest.  Its first key is the Eq. 7 objective beyond the fixed f_i(lo_i) terms, so the
    primary criterion is OptPerf itself; the rest is the canonical tie-break."""
    _check_models(nodes, comm)
    n = len(nodes)
    lo, cap = _bounds(n, B, lo, cap)
    best = None
    best_b = None
    ranges = [range(lo[i], cap[i] + 1) for i in range(n - 1)]
    for head in itertools.product(*ranges):
        last = B - sum(head)
        if not (lo[n - 1] <= last <= cap[n - 1]):
            continue
        b = list(head) + [last]
        keys = sorted(((node_time(nodes[i], comm, float(j)), i)
                       for i in range(n) for j in range(lo[i] + 1, b[i] + 1)), reverse=True)
        if best is None or keys < best:
            best, best_b = keys, b
    return best_b, cluster_time(nodes, comm, best_b)


def round_paper(b_real, B: int):
    """round the relaxed split to integers (largest remainder, ties to lower index)."""
    fl = [math.floor(x) for x in b_real]
    rem = [(x - f, -i) for i, (x, f) in enumerate(zip(b_real, fl))]
    short = B - sum(fl)
    order = sorted(range(len(b_real)), key=lambda i: rem[i], reverse=True)
    out = list(fl)
    for t in range(short):
        out[order[t]] += 1
    return out


def warmup_split(t_sample, B: float):
    """Eq. 8: b_i = (sum_j t_j / t_i) * (sum_l sum_j t_j / t_l)^{-1} * B."""
    tot = sum(t_sample)
    w = [tot / t for t in t_sample]
    norm = sum(w)
    return [wi / norm * B for wi in w]
