"""Oracle: event-driven bucket pipeline of §3.2.3 -- an independent pin for Eq. 5-7.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:169-182 (§3.2.3): gradients are split into buckets; bucket j of every node starts syncing
when all nodes have it ready and the previous bucket's sync is done; only the last bucket (T_u)
is never overlapped; the first bucket is ready at syncStart_i = a_i + gamma P_i (Eq. 4) and the
remaining buckets are "evenly distributed in the rest of gradient computing time and communication
time": ready times evenly spaced over the remaining (1 - gamma) P_i, T_o split evenly over
the first N_b - 1 bucket syncs.
"""
from __future__ import annotations


def simulate(nodes, comm, b, n_buckets: int = 8) -> float:
    """Return the end of the last bucket's synchronisation (the batch time)."""
    assert n_buckets >= 2
    gamma, t_o, t_u = comm
    n = len(nodes)
    ready = []
    for i in range(n):
        q, s, k, m = nodes[i]
        a = q * b[i] + s
        P = k * b[i] + m
        first = a + gamma * P
        ready.append([first + j * (1.0 - gamma) * P / (n_buckets - 1) for j in range(n_buckets)])
    end = 0.0
    for j in range(n_buckets):
        start = max(max(ready[i][j] for i in range(n)), end)
        end = start + (t_o / (n_buckets - 1) if j < n_buckets - 1 else t_u)
    return end
