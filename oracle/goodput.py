"""Oracle: adaptive total batch selection by goodput.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:141-143 (§2.2): the gradient noise scale predicts the statistically efficient batch; Pollux's
*goodput* = system throughput x statistical efficiency modelled by the GNS.  The efficiency form is
Pollux's, (B_noise + B0) / (B_noise + B) relative to the initial batch B0 (reading Q27; the paper
defers to Pollux).  Throughput at total batch B = B / OptPerf(B) (Eq. 7 at the integer split).
B_noise = S / G of exponential moving averages of G and S taken separately (reading Q26; P:343
notes the ratio estimator is biased).
"""
from __future__ import annotations

from . import optsplit


def efficiency(B, B0, B_noise):
    return (B_noise + B0) / (B_noise + B)


def goodput(nodes, comm, B, B0, B_noise):
    _, T = optsplit.int_split_greedy(nodes, comm, B)
    return B / T * efficiency(B, B0, B_noise), T


def choose_batch(nodes, comm, candidates, B0, B_noise):
    """Definition: evaluate every candidate, return the argmax (first on ties)."""
    best, best_g = None, -1.0
    for B in candidates:
        g, _ = goodput(nodes, comm, B, B0, B_noise)
        if g > best_g:
            best, best_g = B, g
    return best


class Ema:
    def __init__(self, decay=0.9):
        self.decay, self.G2, self.trS, self.count = decay, 0.0, 0.0, 0

    def update(self, G2, trS):
        if not G2 > 0.0:
            return
        if self.count == 0:
            self.G2, self.trS = G2, trS
        else:
            self.G2 = self.decay * self.G2 + (1 - self.decay) * G2
            self.trS = self.decay * self.trS + (1 - self.decay) * trS
        self.count += 1

    @property
    def B_noise(self):
        return self.trS / self.G2
