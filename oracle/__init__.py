"""fp64 CPU ORACLE for the DisagFusion DiT stage and its stage handoff.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or execute anything here.  The
product path (paper_2605_25550_b200) never imports it and shares no code with it:
the two meet only through synth/ (seeded inputs and shapes, no method
arithmetic).  Every function cites the PAPER.md passage or DESIGN.md reading it
follows.

Parity status per function (pins in tests/test_oracle_*.py):
  philox       pinned: Random123 known-answer vectors
  params       pinned: uniform-recipe invariants (range, exactness, moments)
  dit.sigmas   pinned: worked values S=4, shifts 1/3/5 (closed form)
  dit.euler    pinned: constant / linear / rectified-flow fields (closed forms)
  dit.attention pinned: brute-force loop softmax, N_kv=1, equal logits
  dit.rope3    pinned: pair-norm, relative-position, identity at origin
  dit.rms_norm pinned: scale invariance, unit rms
  dit.patchify pinned: round trip, hand-indexed elements
  dit.sinusoid pinned: t=0 closed form
  dit.block    pinned: adaLN-zero identity, loop re-derivation on a tiny case
  dit (full composition) — parity unpinned by the paper (no printed values);
               rests on the per-component pins and the vacuity guard
  stages.encoder / decoder — stand-ins (R17); decoder pinned by pixel-shuffle
               index check; encoder composition parity unpinned
  capacity.qps / plan  pinned: the paper's QPM points
  capacity.payload_hash pinned: splitmix64 published first output, chunk additivity
  fp8 (NEXT-4, R28) pinned: E4M3 closed forms, 256-code round trip, ties-to-even,
               saturation, torch float8_e4m3fn cast, brute-force GEMM
"""
