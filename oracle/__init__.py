"""FourierSMT fp64 CPU oracle — TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT.

This package is a plain, slow, obviously-correct CPU implementation of what the
hot path of FourierSMT (arXiv 2603.22877, /root/reference/PAPER.md) computes.
It exists only to prove the CUDA path right. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import, call or execute anything under ``oracle/``. The
product path (``paper_2603_22877_b200``) never imports it and fails loudly when
its CUDA library is missing.

It shares no code with the CUDA path (own parser, own BDD builder, own Philox,
own arithmetic); the only code both sides use is the seeded input generator
package ``fsmt_gen`` which holds none of the method's arithmetic.

Citation convention: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n.
Every reading of an ambiguous/garbled passage is listed in DESIGN.md §3
("Readings") under the R-ids used in the module docstrings below.

Modules
-------
hsmt        HSMT text -> Formula (atoms canonicalised)
semantics   exact fp64 atom / constraint evaluation, slot order (R5, R6, R22)
smoothing   Eq.7 d_i(b) and its gradient P:1326-1327 (R2)
expectation E_c by vertex enumeration (Eq.8 / Lemma P:812-827), sparse xWFE (Cor.1),
            Poisson-binomial count DP for symmetric kinds
objective   C(a,b) = sum_c w_c E_c (Eq.10, Alg.F) and its gradient
philox      Philox4x32-10 counter-based generator (R17, R20)
solve       Alg.2 + Alg.1 step by step
robdd       structure-only ROBDD from a truth table, canonical numbering (Def.2, R7)
bruteforce  exhaustive SAT with exact Fourier-Motzkin (Thm.1 pins)

Parity status: every function above is pinned by tests/test_oracle_*.py
against values the paper prints, closed forms, invariants, or brute force.
The full solve trajectory is "parity unpinned" beyond soundness.
"""
