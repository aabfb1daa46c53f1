"""Host side of the end-to-end transport encodings (no GPU): the weight-stack delta encoding
(fcn.delta_stack, rebuilt on the device by zk_undelta_i8) is lossless, picks the smallest slot stride whose
differences fit int8, and declines stacks it cannot encode."""
import numpy as np
import pytest

from paper_2307_16273_b200 import fcn as dfcn


def rebuild(ds):   # the device rule of zk_undelta_i8, in numpy
    base = ds.base.numpy().astype(np.int32)
    out = np.zeros(ds.shape, np.int32)
    out[:ds.L] = base
    d = ds.delta.numpy().astype(np.int32) if ds.delta is not None else None
    for s in range(ds.L, ds.n_real):
        out[s] = out[s - ds.L] + d[s - ds.L]
    return out


@pytest.mark.parametrize("L", [1, 3, 7])
def test_delta_stack_roundtrip(L):
    rng = np.random.default_rng(L)
    N, n_real, shape = 16, 14, (8, 12)
    a = np.zeros((N,) + shape, np.int32)
    a[:L] = rng.integers(-4096, 4096, (L,) + shape)
    for s in range(L, n_real):   # a few quantisation steps per "training step"
        a[s] = a[s - L] + rng.integers(-3, 4, shape) * (rng.random(shape) < 0.05)
    ds = dfcn.delta_stack(a, n_real, pin=False)
    assert ds is not None and ds.L == L
    assert ds.numel() == L * 96 * 2 + (n_real - L) * 96
    assert np.array_equal(rebuild(ds), a)


def test_delta_stack_declines():
    rng = np.random.default_rng(0)
    a = rng.integers(-30000, 30000, (8, 4, 4)).astype(np.int32)      # unrelated slots: no stride works
    assert dfcn.delta_stack(a, 8, pin=False) is None
    b = np.zeros((4, 4, 4), np.int32)
    b[0, 0, 0] = 1 << 16                                              # first slot beyond int16
    assert dfcn.delta_stack(b, 4, pin=False) is None
    c = np.zeros((4, 3, 3), np.int32)                                 # slot size not a multiple of 4
    assert dfcn.delta_stack(c, 4, pin=False) is None
