"""Oracle: the measured-model loop of PAPER.md §4.5.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* fit_linear     -- P:385-388: from >= 2 local batch sizes fit a_i = q_i b + s_i, P_i = k_i b + m_i
                    (least squares written out: slope = Sxy/Sxx, intercept = ybar - slope xbar).
* ivw            -- Eq. 12: gamma = sum_i (gamma_i / s_i^2) / sum_i (1 / s_i^2), with
                    gamma_i the node's mean observation and s_i^2 the sample variance of its
                    observations (reading Q22 of DESIGN.md).
* comm time      -- P:406: T = min_i T_i.
* plan           -- epoch 0 even split, epoch 1 Eq. 8, then OptPerf from the
                    learned models ("as early as the third epoch").
"""
from __future__ import annotations

import math

from . import optsplit


def fit_linear(x, y):
    n = len(x)
    if n < 2:
        raise ZeroDivisionError("need >= 2 points")
    mx = sum(x) / n
    my = sum(y) / n
    sxx = sum((xi - mx) * (xi - mx) for xi in x)
    sxy = sum((xi - mx) * (yi - my) for xi, yi in zip(x, y))
    if sxx == 0.0:
        raise ZeroDivisionError("all x equal")
    slope = sxy / sxx
    return slope, my - slope * mx


def ivw(estimates, variances):
    zero = [e for e, v in zip(estimates, variances) if v == 0.0]
    if zero:
        return sum(zero) / len(zero)
    num = sum(e / v for e, v in zip(estimates, variances))
    den = sum(1.0 / v for v in variances)
    return num / den


def sample_variance(xs):
    m = sum(xs) / len(xs)
    return sum((x - m) * (x - m) for x in xs) / (len(xs) - 1)


class Analyzer:
    """Keeps each node's observations (b, a, P, gamma, t_o, t_u); plans each epoch."""

    def __init__(self, n):
        self.n = n
        self.obs = [[] for _ in range(n)]

    def observe(self, node, it, b, a, P, gamma, t_o, t_u):
        self.obs[node].append((b, a, P, gamma, t_o, t_u, it))

    def models(self):
        nodes, gm, gv, to, tu = [], [], [], [], []
        for v in self.obs:
            xs = [float(o[0]) for o in v]
            q, s = fit_linear(xs, [o[1] for o in v])
            k, m = fit_linear(xs, [o[2] for o in v])
            tiny = 1e-12
            nodes.append((max(q, tiny), max(s, 0.0), max(k, tiny), max(m, 0.0)))
            g = [o[3] for o in v]
            gm.append(sum(g) / len(g))
            gv.append(sample_variance(g) if len(g) >= 2 else None)
            to.append(sum(o[4] for o in v) / len(v))
            tu.append(sum(o[5] for o in v) / len(v))
        pairs = [(e, w) for e, w in zip(gm, gv) if w is not None]
        gamma = ivw([p[0] for p in pairs], [p[1] for p in pairs]) if pairs else sum(gm) / len(gm)
        gamma = min(max(gamma, 0.0), 0.999999)
        # T = min_i T_i per iteration, averaged over the iterations all nodes reported
        iters = sorted({o[6] for o in self.obs[0]})
        mins_o, mins_u = [], []
        for it in iters:
            per = [[o for o in v if o[6] == it] for v in self.obs]
            if all(per):
                mins_o.append(min(o[4] for p in per for o in p))
                mins_u.append(min(o[5] for p in per for o in p))
        if mins_o:
            t_o, t_u = sum(mins_o) / len(mins_o), sum(mins_u) / len(mins_u)
        else:
            t_o, t_u = min(to), min(tu)
        return nodes, (gamma, max(t_o, 0.0), max(t_u, 0.0))

    def plan(self, B, cap=None):
        n = self.n
        distinct = [len({o[0] for o in v}) for v in self.obs]
        if all(d >= 2 for d in distinct):
            nodes, comm = self.models()
            b, T = optsplit.int_split_greedy(nodes, comm, B, cap=cap)
            return {"b": b, "T_pred": T, "phase": 2}
        if all(self.obs):
            ts = []
            for v in self.obs:
                bl = v[-1][0]
                sel = [(o[1] + o[2]) / o[0] for o in v if o[0] == bl]
                ts.append(sum(sel) / len(sel))
            b = optsplit.round_paper(optsplit.warmup_split(ts, B), B)
            b = [max(x, 1) for x in b]
            s, i = sum(b), 0
            while s > B and i < 4 * n:
                if b[i % n] > 1:
                    b[i % n] -= 1
                    s -= 1
                i += 1
            phase = 1
        else:
            b = [B // n + (1 if i < B % n else 0) for i in range(n)]
            phase = 0
        if cap is not None:
            excess = 0
            for i in range(n):
                if b[i] > cap[i]:
                    excess += b[i] - cap[i]
                    b[i] = cap[i]
            for i in range(n):
                give = min(cap[i] - b[i], excess)
                b[i] += give
                excess -= give
        return {"b": b, "T_pred": math.nan, "phase": phase}
