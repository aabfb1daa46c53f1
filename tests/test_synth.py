"""The seeded input generators (no method arithmetic): the torch generator used on the GPU box for
large / per-rank inputs is bit-identical to the numpy one every oracle test uses."""
import numpy as np

from synth.prng import uniform_bits, uniform_range, uniform_range_torch


def test_torch_generator_matches_numpy():
    for tid, lo, hi, off in [(21, -(1 << 15), 1 << 15, 0), (22, -(1 << 15), 1 << 15, 987654),
                             (11, -(1 << 31), 1 << 31, 0), (3, 0, 2, 5)]:
        a = uniform_range_torch(230716273, tid, 3000, lo, hi, "cpu", offset=off, chunk=1024).numpy()
        bits = (hi - lo).bit_length() - 1
        b = uniform_bits(230716273, tid, 3000, lo, bits, offset=off).astype(np.int32)
        assert (a == b).all()
    full = uniform_range(230716273, 21, (4096,), -(1 << 15), 1 << 15)
    halves = [uniform_range_torch(230716273, 21, 2048, -(1 << 15), 1 << 15, "cpu", offset=o).numpy() for o in (0, 2048)]
    assert (np.concatenate(halves) == full).all()   # rank slices of a sharded statement
