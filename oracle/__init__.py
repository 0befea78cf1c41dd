"""CPU oracle for the Cannikin data-parallel hot path (arXiv 2402.05302).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from this package.  The product
path (``paper_2402_05302_b200`` and the CUDA library) never imports, calls or links it, and the
oracle imports nothing from the product path: the two share no code.  Inputs come from
``cannikin_synth`` (random draws only, no arithmetic of the method).

Plain, slow, obviously-correct NumPy float64, following PAPER.md in its own order and notation:

* ``aggregate``  -- Eq. 9 weighted aggregation g = sum_i r_i g_i, r_i = b_i / B and the
  squared norms ||g_i||^2, ||g||^2 the GNS needs (Eq. 10 inputs).
* ``gns``        -- Eq. 10 local estimates, Theorem 1 weights, B_noise = S/G.
* ``optsplit``   -- per-node time (Eq. 3-7), the real r_opt (equal finish times, §3.3 /
  App. A), the exact integer split, brute force, the paper's rounding
   and the Eq. 8 warm-up split.
* ``pipeline``   -- the event-driven bucket pipeline of §3.2.3, an independent pin for the
  closed-form per-node time.

Every function is pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``) against values printed in
the paper / SPEC.md worked examples, closed forms, invariants and brute force.  Functions with no
such pin say "parity unpinned" in their docstring (none at present).
"""
