"""oracle/ -- TEST INFRASTRUCTURE.  A plain, slow, obviously correct CPU
implementation (float64 numpy + a plain-C double codec) of what the VaPr
rollout hot path computes, written from PAPER.md and the readings listed in
DESIGN.md §3.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import or execute anything here.  The product
path (paper_2310_07854_b200/) never imports it and shares no code with it;
both consume the seeded inputs of workloads/ only.

Modules:
  codec       ExMy quantize/dequantize (C formula + numpy enumeration), packing
  formats     the 21-format space and the search-space arithmetic
  kinematics  Panda FK / BK in float64
  collision   box SDF, smooth hinge, world (discrete/swept) and self costs
  rollout     the staged FK -> world -> self -> aggregate -> BK dataflow
  lbfgs       L-BFGS two-loop direction, N-scale line search, history (N1)
Parity status of each function is listed in DESIGN.md §4 (all pinned; the
"3.5x-4.4x tensor size reduction" figure of PAPER.md:316 is parity unpinned
and is not computed here).
"""
