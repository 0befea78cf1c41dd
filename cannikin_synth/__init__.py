"""Seeded synthetic-input generators shared by the oracle tests, the CUDA-path tests and bench.py.

This module holds NO arithmetic of the method (no weighted sum, no norm, no GNS estimator, no
split solver).  It only draws the random inputs the method is applied to, following the input
recipe of DESIGN.md §3:

* gradients: ``g_i = G + sqrt(trS / (N * b_i)) * eps_i`` -- the distribution of the mean of b_i
  per-sample gradients drawn from N(G, (trS/N) I) (Eq. 1; §4.4).
  ``G`` is a fixed random direction scaled so that ``||G||^2 = G2``.
* value set V2 ("layered"): per-2^16-element block scale 10^U(-4,0) plus 1e-3 of x100 outliers.
* value set V3: special cases (zeros, identical g_i).
* the cast to fp32 / bf16 (round-to-nearest-even) produces the *inputs of record*: every
  consumer (oracle and CUDA path) starts from exactly these bits.
* random node/comm models for the opt_split fixtures.

bf16 values are carried as ``numpy.uint16`` bit patterns (numpy has no bfloat16 dtype).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "rank_generators",
    "f32_to_bf16_bits",
    "gns_gradients",
    "layered_gradients",
    "per_sample_gradients",
    "random_cluster",
    "device_gns_gradients",
]


def rank_generators(seed: int, n: int) -> list[np.random.Generator]:
    """n+1 independent PCG64 substreams: index 0 draws G, index 1+i draws rank i's noise."""
    ss = np.random.SeedSequence(seed)
    return [np.random.Generator(np.random.PCG64(c)) for c in ss.spawn(n + 1)]


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (round-to-nearest-even) and return the uint16 bits.

    This is the input cast (the "inputs of record" step), not part of the method.
    NaN is not produced by the generators, so no NaN special-casing is needed.
    """
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    rounded = (u + 0x7FFF + lsb) >> 16
    return rounded.astype(np.uint16)


def _cast(x64: np.ndarray, dtype: str) -> np.ndarray:
    x32 = x64.astype(np.float32)
    if dtype == "f32":
        return x32
    if dtype == "bf16":
        return f32_to_bf16_bits(x32)
    raise ValueError(f"unknown dtype {dtype!r}")


def gns_gradients(n: int, N: int, b, *, G2: float = 1.0, trS: float = 100.0, seed: int = 0,
                  dtype: str = "f32") -> list[np.ndarray]:
    """V1: per-rank mean gradients with known ||G||^2 = G2 and tr(Sigma) = trS.

    Returns n arrays of N elements (float32, or uint16 bf16 bits).
    """
    b = [int(x) for x in b]
    assert len(b) == n and all(x >= 1 for x in b)
    gens = rank_generators(seed, n)
    if N == 0:
        return [_cast(np.zeros(0), dtype) for _ in range(n)]
    z = gens[0].standard_normal(N)
    G = z * np.sqrt(G2 / np.dot(z, z))
    out = []
    for i in range(n):
        sd = np.sqrt(trS / (N * b[i]))
        out.append(_cast(G + sd * gens[1 + i].standard_normal(N), dtype))
    return out


def layered_gradients(n: int, N: int, *, seed: int = 0, dtype: str = "f32",
                      block: int = 1 << 16, outlier_frac: float = 1e-3) -> list[np.ndarray]:
    """V2: precision stress -- per-block magnitudes spanning 4 decades plus x100 outliers."""
    gens = rank_generators(seed, n)
    nblk = max(1, -(-N // block))
    scales = 10.0 ** gens[0].uniform(-4.0, 0.0, size=nblk)
    out = []
    for i in range(n):
        g = gens[1 + i].standard_normal(N) * np.repeat(scales, block)[:N]
        k = int(outlier_frac * N)
        if k:
            idx = gens[1 + i].choice(N, size=k, replace=False)
            g[idx] *= 100.0
        out.append(_cast(g, dtype))
    return out


def per_sample_gradients(b, d: int, *, G2: float = 1.0, trS: float = 100.0, seed: int = 0):
    """Per-sample gradients x_{i,j} ~ N(G, (trS/d) I) in float64, as a list of (b_i, d) arrays.

    Used for the exactness pin "Eq. 9 of per-node means == mean of all B per-sample gradients"
     and for Monte-Carlo pins of the §4.4 identity.
    """
    n = len(b)
    gens = rank_generators(seed, n)
    z = gens[0].standard_normal(d)
    G = z * np.sqrt(G2 / np.dot(z, z))
    sd = np.sqrt(trS / d)
    return G, [G + sd * gens[1 + i].standard_normal((int(b[i]), d)) for i in range(n)]


def random_cluster(rng: np.random.Generator, n: int, *, scale: float = 1.0):
    """Random node models (q, s, k, m) and a comm model (gamma, t_o, t_u) for opt_split fixtures.

    Magnitudes follow the shape of the paper's setting (§3.2, Eq. 3-4): per-sample times of
    0.1-10 ms, fixed costs of 1-100 ms, gamma in (0, 0.5), T_o comparable to the backprop time so
    that both bottleneck patterns occur.
    """
    nodes = []
    for _ in range(n):
        q = float(rng.uniform(1e-4, 5e-3)) * scale
        k = float(rng.uniform(1e-4, 1e-2)) * scale
        s = float(rng.uniform(1e-3, 1e-1))
        m = float(rng.uniform(1e-3, 1e-1))
        nodes.append((q, s, k, m))
    gamma = float(rng.uniform(0.0, 0.5))
    t_o = float(rng.uniform(0.0, 0.4))
    t_u = float(rng.uniform(0.0, 0.1))
    return nodes, (gamma, t_o, t_u)


def device_gns_gradients(n: int, N: int, b, *, G2: float = 1.0, trS: float = 100.0, seed: int = 0,
                         dtype: str = "f32", device="cuda", ranks=None):
    """V1 recipe generated directly on the GPU with torch (for sizes the host cannot draw fast).

    Returns a list of device tensors (torch.float32 or torch.bfloat16).  The tensors ARE the inputs
    of record: any oracle comparison downloads these exact bits.  ``ranks`` selects which ranks
    to materialise (default: all) so that a multi-GPU rank can draw only its own gradient.
    """
    import torch

    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed) * 1000003 + 17)
    z = torch.randn(N, generator=gen, device=device, dtype=torch.float32)
    G = z * torch.sqrt(torch.tensor(G2, device=device) / torch.dot(z, z))
    out = []
    for i in range(n) if ranks is None else ranks:
        gi = torch.Generator(device=device)
        gi.manual_seed(int(seed) * 1000003 + 1009 * (i + 1))
        eps = torch.randn(N, generator=gi, device=device, dtype=torch.float32)
        sd = float(np.sqrt(trS / (max(N, 1) * int(b[i]))))
        out.append((G + sd * eps).to(tdt))
        del eps
    return out


def simulate_iteration(nodes, comm, b, rng: np.random.Generator, cv: float = 0.0,
                       gamma_sd=None):
    """Noisy timing telemetry of one iteration of a cluster with TRUE models (q, s, k, m) and comm
    model (gamma, T_o, T_u), for the measured-model loop tests (inputs only, no estimator):
      a_i, P_i   = Eq. 3 times x lognormal noise with coefficient of variation cv (mean 1)
      gamma_i    = gamma + N(0, gamma_sd[i])    (node-specific measurement noise, fig:overlapratio)
      T_o_i, T_u_i = T_o, T_u + the time node i waits for the slowest node to reach the first
                   bucket ("each node reports different T_i ... because of the
                   wait-for-synchronization time"); the slowest node waits 0.
    Returns a list of dicts, one per node."""
    gamma, t_o, t_u = comm
    n = len(nodes)
    if gamma_sd is None:
        gamma_sd = [0.0] * n

    def ln():
        if cv <= 0.0:
            return 1.0
        s2 = np.log(1.0 + cv * cv)
        return float(np.exp(rng.normal(-0.5 * s2, np.sqrt(s2))))

    a = [(nodes[i][0] * b[i] + nodes[i][1]) * ln() for i in range(n)]
    P = [(nodes[i][2] * b[i] + nodes[i][3]) * ln() for i in range(n)]
    start = [a[i] + gamma * P[i] for i in range(n)]
    last = max(start)
    out = []
    for i in range(n):
        wait = last - start[i]
        out.append({"a": a[i], "P": P[i],
                    "gamma": gamma + (float(rng.normal(0.0, gamma_sd[i])) if gamma_sd[i] > 0 else 0.0),
                    "t_o": t_o + wait, "t_u": t_u + wait})
    return out
