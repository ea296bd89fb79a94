"""CPU oracle for the BoostCom BGV word-wise comparison hot path (arXiv 2407.07308).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_2407_07308_b200``) never imports it and shares no code with it.

The oracle is a plain, slow, obviously-correct implementation of what the path
computes, written from PAPER.md (cited as ``P:<line>``) and the readings listed
in DESIGN.md §3 (cited as ``R<k>``):

* ``nt``       -- primality, NTT-friendly prime search, roots of unity, CRT.
* ``cyclo``    -- Phi_m over Z, Z_m^*, schoolbook products mod (q, Phi_m), naive
                  evaluation at the primitive m-th roots (the "evaluation form"),
                  and a literal step-by-step BluesteinNTT used only to
                  pin the paper's transform description against the naive DFT.
* ``slots``    -- the plaintext slot algebra F_p[x]/Phi_m = prod F_{p^D}; encode /
                  decode; integer <-> digit encoding (Table 3).
* ``prng``     -- the counter-based sampler both sides implement (R7).
* ``bgv``      -- keygen / encrypt / decrypt / tensor / hybrid key switching /
                  modulus switching / automorphisms, all in coefficient form with
                  naive big-integer CRT.
* ``circuits`` -- digit LT/EQ polynomials (interpolation), Paterson-Stockmeyer and
                  bivariate schedules, Frobenius digit extraction, lexicographic
                  combination (ShiftMul/ShiftAdd), select/min/max, slot
                  compaction.

Functions whose result has no independent pin say "parity unpinned" in their
docstring.
"""
