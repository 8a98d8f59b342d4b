"""paper_2002_02885_b200 — B200-native pack primitive (arxiv 2002.02885).

Drop-in for the reference's `packtrain` pack path:

    from paper_2002_02885_b200 import packing, tuner, data
    packed = packing.dedup_inputs(packing.pack_models([a, b]))
    losses = packing.packed_step(packed, datasets)

`packing` / `tuner` / `data` / `engine` mirror the reference modules of the
same names; the step runs in libpk_b200.so (hand-written sm_100a kernels,
C-ABI in include/packtrain_b200.h).
"""
__version__ = "0.1.0"
