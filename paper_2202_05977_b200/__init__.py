"""B200-native kernel-map decoder + per-pixel filter + kernel fusion
(arXiv 2202.05977, "weight sharing kernel prediction", reconstruction phase).

The product is libkmd.so (C ABI, include/kmd.h) built from ``csrc/``;
``kmd`` is its thin Python binding and ``inputs`` the seeded synthetic input
generator.  Importing the package does not load the CUDA library; the first
call does, and raises if it is missing (there is no CPU fallback).
"""
from . import inputs  # noqa: F401
from .inputs import PAPER_SIZES, make_inputs  # noqa: F401

