"""B200-native (sm_100a) hot path of 6Bit-Diffusion (arxiv 2603.18742): DMPQ + TDC.

The product is libdmpq.so (C ABI in include/dmpq.h); this package is its Python
binding (paper_2603_18742_b200.dmpq), the seeded synthetic-input generators
(synth), the block-step driver (block) and token sharding (shard).
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"
