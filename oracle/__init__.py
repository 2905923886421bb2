"""fp64 CPU ORACLE for the DisagFusion DiT stage and its stage handoff.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or execute anything here.  The
product path (paper_2605_25550_b200) never imports it and shares no code with it:
the two meet only through synth/ (seeded inputs and shapes, no method
arithmetic).  Every function cites the PAPER.md passage or DESIGN.md reading it
follows.

Parity status per function (pins in tests/test_oracle_*.py; every pin
is checked to fail under one-line mutations of the oracle by tools/mutate_oracle.py,
38/38 killed, profiles/r02_oracle_mutations.txt):
  philox       pinned: Random123 known-answer vectors
  params       pinned: uniform-recipe invariants (range, exactness, moments)
  dit.sigmas   pinned: worked values S=4, shifts 1/3/5 (closed form)
  dit.euler    pinned: constant / linear / rectified-flow fields (closed forms)
  dit.attention pinned: brute-force loop softmax, N_kv=1, equal logits
  dit.rope3    pinned: pair-norm, relative-position, identity at origin
  dit.rms_norm pinned: scale invariance, unit rms
  dit.patchify pinned: round trip, hand-indexed elements
  dit.sinusoid pinned: t=0 closed form
  dit.time_embedding pinned: identity-like W_e1/W_e2/W_m closed form at sigma = 0.37 and 0
  dit.text_projection pinned: one-hot W_t1, shifted W_t2 closed form (GELU side, b_t1 inside)
  dit.cross_kv pinned: per-head RMS of K = |g_ck| at any per-head scale, V un-normalised
  dit.head     pinned: shift-only / scale-only hand-indexed outputs
  dit.velocity pinned (wiring): zero-layer DiT = head(patch embed, e) closed form
  dit.block    pinned: adaLN-zero identity; modulation rows 0/1 (uniform self-attention
               closed form), rows 3/4 and the SwiGLU sides (linear / SiLU special cases),
               gates, cross-attention ungated and unmodulated, cross query path closed form
  dit (full composition) -- parity unpinned by the paper (no printed values);
               rests on the per-function pins above and the vacuity guard
  stages.encoder pinned: one-token closed form (SiLU side, residual, gains)
  stages.decoder pinned: pixel-shuffle index check
  capacity.qps / plan  pinned: the paper's QPM points
  capacity.payload_hash pinned: splitmix64 published first output, chunk additivity
  fp8 (NEXT-4, R28) pinned: E4M3 closed forms, 256-code round trip, ties-to-even,
               saturation, torch float8_e4m3fn cast, brute-force GEMM
  fp8.mx_* (NEXT-4, R30 MXFP8) pinned: block-exponent closed form, worked block 1..32
               (ties-to-even), exact round trips, OCP saturation, block independence,
               zero block, torch cast of the scaled values, half-quantum error bound,
               brute-force GEMM
  dit_fp8 (NEXT-4, R29) pinned: per-row quantiser closed forms (amax-448 row, zero row,
               power-of-two scaling); wiring = dit.block exactly under identity quantisers
  dit_fp8.mx_act / mx_weight (R31) pinned: blocks along K per output column, row independence
  dit_fp8.qk_scale / qk_quant (R32) pinned: the worst-case component bound (lands in
               (224, 448]), power of two, e4m3 relative precision of typical components
  dit_fp8.v_quant (R33) pinned: exact round trip of scaled codes, power-of-two scale
               (amax 100 -> 96 by ties-to-even), half-quantum relative error
"""
