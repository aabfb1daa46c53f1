"""Seeded synthetic input generators shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the proving method (no field arithmetic, no
eq/MLE, no sumcheck, no zkReLU relations).  It produces plain integer tensors
from a counter-based PRNG (SURVEY.md §8(d) "Synthetic-data rules") and the
quantized FCN training trace that the prover consumes as its input (PAPER.md
L321, Protocol 1 line 2: "Prover executes training steps" — training is the
prover's input, not part of the proof).
"""
from .prng import DATA_SEED, fs_seed, uniform_bits, uniform_range  # noqa: F401
