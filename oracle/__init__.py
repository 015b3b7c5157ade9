"""Oracle for the Acc-SpMM hot path (arXiv 2501.09251) -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations of what the hot path
computes, each function citing the PAPER.md / SPEC.md passage it follows
(``P:n`` = /root/reference/PAPER.md line n, ``S:n`` = SPEC.md line n,
``SURVEY §8(c)`` = the reading adopted where the paper is silent).

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import, call, link or execute
anything under ``oracle/``.  The oracle shares no code with the product
package ``paper_2501_09251_b200`` and never imports it; the product never
imports the oracle.  Inputs come from the method-free ``gen`` package.

Modules and pins:

* ``rounding``  -- rho: TF32 round-to-nearest-away and FP16 RNE.
                   Pinned by an fp64 closed form of round-half-away-from-zero and
                   numpy's IEEE float16 cast; on the GPU box by the hardware
                   ``cvt.rna.tf32.f32`` over all 2^32 bit patterns.
* ``spmm``      -- FP64 CSR SpMM + bound (C, spmm_oracle.c).  Pinned by dense
                   GEMM brute force, SPEC S:86-88 examples, integer exactness.
* ``bittcf``    -- BitTCF encode/decode/byte formulas.  Pinned by the
                   P:253 byte formula, worked fixtures, decode round trip.
* ``balance``   -- IBD Eq. (3), Eq. (4), the unit schedule.  Pinned by
                   S:418-419 / S:427 worked values and coverage invariants.
* ``partition`` -- nnz-balanced window ranges (BASELINE north_star).  Pinned by
                   brute force.
* ``reorder``   -- Algorithm 1.  A heuristic: parity is pinned only
                   by invariants (bijection, Q/dQ closed forms, clique contiguity,
                   MeanNNZTC gain) -- "parity unpinned" for the exact ordering.
"""
