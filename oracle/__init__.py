"""QTIP CPU oracle (arXiv 2406.11235) -- TEST INFRASTRUCTURE ONLY.

This package is a plain, slow, obviously-correct float64 / exact-integer
re-statement of what the QTIP inference path computes, written from
PAPER.md.  It exists to *check* the CUDA library, never to serve it:

  * only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import or execute it;
  * it shares no code, tables, constants generators or pre/post-processing
    with ``paper_2406_11235_b200`` (the product), and neither imports the
    other.  The only shared module is ``synth`` (seeded random inputs, no
    method arithmetic).

Citations ``P:<line>`` point at /root/reference/PAPER.md (section / algorithm
/ equation named beside each).  Every function is pinned by a ``-m "not gpu"``
test against something other than itself (paper values, closed forms,
invariants, brute force); see tests/test_oracle_*.py and DESIGN.md §3.

Modules
  trellis   bitshift-trellis edge rule, windows, logical pack/unpack
  codes     1MAD / 3INST / HYB node-value codes (Alg. 1-3), k-means LUT
  hadamard  Sylvester + Paley-I Hadamard matrices
  rht       random Hadamard transform in/out, incoherence mu
  gemv      dense decode of a packed matrix + float64 y = W x
  viterbi   Viterbi DP, constrained DP + Alg. 4 tail-biting,
            brute force.  DP core in plain C (viterbi.c).
  ldlq      BlockLDLQ with QTIP rounding (Algorithm 5): T_y-block LDL, error feedback,
            synthetic AR(1) proxy Hessians.
"""
