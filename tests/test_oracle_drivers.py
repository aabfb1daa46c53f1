"""Oracle drivers: golden regression (files written by scripts/make_golden.py from
the oracle only), determinism, and the FCN family driver on a tiny trace."""
import json
import os

import numpy as np

from synth import fcn
from synth.prng import fs_seed

HERE = os.path.dirname(os.path.abspath(__file__))


def test_c1_golden(oracle_lib):
    from oracle import drivers
    g = json.load(open(os.path.join(HERE, "golden", "c1_transcript.json")))
    res = drivers.c1_prove()
    assert hex(res["claim"]) == g["claim"]
    assert [[hex(v) for v in row] for row in res["msgs"]] == g["msgs"]
    assert [hex(v) for v in res["finals"]] == g["finals"]
    assert res["state"].hex() == g["final_state"]
    assert len(res["msgs"]) == 6 and all(len(r) == 3 for r in res["msgs"])   # m = logN + logD2 = 0 + 6, deg 2


def test_relu_small_golden(oracle_lib):
    from oracle import drivers
    g = json.load(open(os.path.join(HERE, "golden", "relu_small.json")))
    res = drivers.c2_prove(D=64, seed_name="C2-small")
    assert [hex(v) for v in res["claims"]] == g["claims"]
    assert [[hex(v) for v in row] for row in res["msgs"]] == g["msgs"]
    assert res["state"].hex() == g["final_state"]


def test_c5_small_verifies(oracle_lib):
    from oracle import drivers
    O = oracle_lib
    A, B = drivers.c5_inputs(8)
    tr = O.Transcript(fs_seed("C5-test"))
    res = drivers.single_sumcheck_i32(tr, A, B)
    tv = O.Transcript(fs_seed("C5-test"))
    tv.absorb("c5/hdr", (8).to_bytes(4, "little"))
    assert tv.challenges("c5/w", 8) == res["w"]
    P = O.P
    ta = [int(v) % P for v in A]
    tb = [int(v) % P for v in B]
    assert O.sumcheck_verify(tv, 8, 8, 2, res["w"], res["claim"], res["msgs"], res["finals"], [ta, tb]) == 0


def test_fcn_family_driver_tiny(oracle_lib):
    from oracle import drivers
    shape = fcn.tiny_shape(steps=2, layers=3, width=8, batch=4, din=8, dout=4)
    trace = fcn.generate_trace(shape, x_bits=4, w_bits=4, y_bits=3)
    fams = fcn.assemble_families(shape, trace)
    names = [f.name for f in fams]
    assert names[0].startswith("ReLU[") and names[1].startswith("F[") and names[-1].startswith("GW[")
    out = drivers.fcn_prove(shape, fams, "tiny")
    assert len(out) == len(fams)
    # the trace's product tensors satisfy the matmul identity at the drawn points
    O = oracle_lib
    for f, res in zip(fams, out):
        if isinstance(f, fcn.MatmulFamily):
            Y = f.Y.reshape(-1)
            assert res["claim"] == O.mle_i32(Y, res["u3"] + res["u1"] + res["w"])
    again = drivers.fcn_prove(shape, fams, "tiny")
    assert [r["state"] for r in again] == [r["state"] for r in out]       # determinism
    # D3d forks: family f's transcript depends only on the window header and the names up to f
    first = drivers.fcn_prove(shape, fams, "tiny", only=2)
    assert [r["state"] for r in first] == [r["state"] for r in out[:2]]
    # the window state is the join of the family states, written out with the transcript primitives
    from synth.prng import fs_seed
    W = O.Transcript(fs_seed("tiny"))
    W.absorb("fcn/hdr", fcn.fcn_header(shape))
    for f in fams:
        W.absorb("fcn/fam", f.name.encode())
        W.challenges("fcn/fork", 1)
    for r in out:
        W.absorb("fcn/join", r["state"])
    assert W.state() == out[-1]["window_state"]
