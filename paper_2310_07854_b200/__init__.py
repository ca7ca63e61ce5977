"""paper_2310_07854_b200 -- B200-native (sm_100a) VaPr rollout hot path.

The product is libvapr.so (C ABI, include/vapr.h) built from csrc/ by
`python -m paper_2310_07854_b200.build`; `binding` is the thin ctypes layer
with the same function names, `rollout` a device-resident runner, `search`
the host VaPr format-search driver (Phase-1 binary search, space reduction,
NSGA-II).  There is no CPU fallback: importing `binding` fails loudly when the
library is missing.
"""
__version__ = "0.1.0"
