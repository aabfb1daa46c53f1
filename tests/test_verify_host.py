"""The host verifiers of libzkdl (D23; verify.cu) on CPU (-m "not gpu").

The verifiers share no code with the oracle; here they are run on the ORACLE's proofs (the GPU
proofs are bit-identical to them, tests/test_gpu_parity.py) and must accept them, end in the oracle
prover's transcript state, and reject tampered proofs at the round the tampering breaks.  The host
transcript is pinned to the oracle's (itself pinned to RFC 7693 vectors, test_oracle_field.py).
"""
import random

import numpy as np
import pytest

from synth.prng import fs_seed, uniform_range

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


@pytest.fixture(scope="module")
def V():
    from paper_2307_16273_b200 import build
    build.build(verbose=False)
    from paper_2307_16273_b200 import verify
    return verify


def u32s(*v):
    return b"".join(int(x).to_bytes(4, "little") for x in v)


def frs(vals):
    return b"".join(int(x).to_bytes(32, "little") for x in vals)


def sc_proof(m, n_eq, K, res):
    return u32s(m, n_eq, K) + frs([res["claim"]]) + frs([v for row in res["msgs"] for v in row]) + frs(res["finals"])


def relu_proof(logD, Q, R, res):
    return u32s(logD, Q, R) + frs(res["claims"]) + frs([v for row in res["msgs"] for v in row]) + frs(res["finals"])


def test_host_transcript_matches_oracle(V, oracle_lib):
    O = oracle_lib
    for seed in (b"\0" * 32, fs_seed("htr")):
        a, b = V.HostTranscript(seed=seed), O.Transcript(seed)
        assert a.state() == b.state()
        for n, tag, msg in ((1, "x", b""), (3, "a/b", b"\x01" * 63), (2, "t" * 40, bytes(range(200)))):
            a.absorb(tag, msg)
            b.absorb(tag, msg)
            assert a.state() == b.state()
            assert a.challenges(tag, n) == b.challenges(tag, n)
            assert a.state() == b.state()


@pytest.mark.parametrize("m,n_eq,K", [(1, 0, 1), (4, 4, 2), (6, 3, 2), (5, 0, 3), (7, 7, 3)])
def test_sumcheck_verifier_on_oracle_proofs(V, oracle_lib, m, n_eq, K):
    O = oracle_lib
    rng = random.Random(11 * m + K)
    tabs = [[rng.randrange(P) for _ in range(1 << m)] for _ in range(K)]
    w = [rng.randrange(P) for _ in range(n_eq)]
    seed = fs_seed(f"vsc-{m}-{n_eq}-{K}")
    T = O.Transcript(seed)
    res = O.sumcheck_prove(T, m, n_eq, tabs, w)
    proof = sc_proof(m, n_eq, K, res)
    H = V.HostTranscript(seed=seed)
    assert V.verify_sumcheck(H, proof, w, shape=(m, n_eq, K)) == res["r"]
    assert H.state() == T.state()
    assert V.verify_sumcheck(V.HostTranscript(seed=seed), proof, w, claim=res["claim"], shape=(m, n_eq, K)) == res["r"]
    assert V.sumcheck_finals(proof) == res["finals"]
    # finals are the MLEs of the tables at r (what a commitment opening would close)
    assert res["finals"] == [O.mle_fr(t, res["r"]) for t in tabs]
    with pytest.raises(V.Rejected) as e:   # another claim
        V.verify_sumcheck(V.HostTranscript(seed=seed), proof, w, claim=(res["claim"] + 1) % P, shape=(m, n_eq, K))
    assert e.value.where == -1
    for t in range(m):                       # one evaluation of round t changed: round t fails
        bad = bytearray(proof)
        o = 44 + 32 * (t * (K + 1))
        bad[o:o + 32] = ((int.from_bytes(bad[o:o + 32], "little") + 1) % P).to_bytes(32, "little")
        with pytest.raises(V.Rejected) as e:
            V.verify_sumcheck(V.HostTranscript(seed=seed), bytes(bad), w, shape=(m, n_eq, K))
        assert e.value.where == t + 1
    bad = bytearray(proof)                   # a final changed: the final identity fails
    bad[-1] ^= 0x01
    with pytest.raises(V.Rejected) as e:
        V.verify_sumcheck(V.HostTranscript(seed=seed), bytes(bad), w, shape=(m, n_eq, K))
    assert e.value.where == -100
    with pytest.raises(ValueError):          # malformed
        V.verify_sumcheck(V.HostTranscript(seed=seed), proof[:-1], w, shape=(m, n_eq, K))
    # the statement's shape is the verifier's: another header is rejected before anything is read
    # (a proof for (m=1, n_eq=0, K=1) passed for any family)
    with pytest.raises(V.Rejected) as e:
        V.verify_sumcheck(V.HostTranscript(seed=seed), proof, w, shape=(m + 1, n_eq, K))
    assert e.value.where == -2
    fake = (u32s(1, 0, 1) if (m, n_eq, K) != (1, 0, 1) else u32s(2, 0, 1)) + frs([5, 2, 3, 4])
    with pytest.raises(V.Rejected) as e:
        V.verify_sumcheck(V.HostTranscript(seed=seed), fake, w, shape=(m, n_eq, K))
    assert e.value.where == -2


def test_hadamard_zero_verifier(V, oracle_lib):
    O = oracle_lib
    m = 6
    A = uniform_range(41, 1, (1 << m,), -(1 << 15), 1 << 15)
    B = uniform_range(41, 2, (1 << m,), -(1 << 15), 1 << 15)
    Y = (A.astype(np.int64) * B).astype(np.int32)
    for bad_at in (None, 5):
        Yx = Y.copy()
        if bad_at is not None:
            Yx[bad_at] += 1
        seed = fs_seed(f"vhd-{bad_at}")
        T = O.Transcript(seed)
        res = O.zero_sumcheck_prove(T, Yx, A, B)
        proof = u32s(m) + frs([v for row in res["msgs"] for v in row]) + frs(res["finals"])
        H = V.HostTranscript(seed=seed)
        if bad_at is None:
            out = V.verify_hadamard_zero(H, proof, m)
            assert out["w"] == res["w"] and out["r"] == res["r"] and H.state() == T.state()
        else:
            with pytest.raises(V.Rejected) as e:
                V.verify_hadamard_zero(H, proof, m)
            assert e.value.where == 1        # the zero claim breaks in the first round


@pytest.mark.parametrize("logD,Q,R", [(4, 16, 16), (6, 8, 8), (5, 12, 4)])
def test_relu_verifier_and_merge(V, oracle_lib, logD, Q, R):
    O = oracle_lib
    lim = 1 << (Q + R - 1)
    Z = uniform_range(42, logD, (1 << logD,), -lim, lim)
    GA = uniform_range(42, logD + 9, (1 << logD,), -lim, lim)
    seed = fs_seed(f"vrelu-{logD}-{Q}-{R}")
    T = O.Transcript(seed)
    res = O.relu_prove(T, Z, GA, Q, R)
    mg = O.relu_merge(T, Z, GA, Q, R, res["point"], res["finals"])
    proof = relu_proof(logD, Q, R, res)
    H = V.HostTranscript(seed=seed)
    v = V.verify_relu(H, proof, (logD, Q, R))
    assert v["point"] == res["point"] and v["claims"] == res["claims"] and v["finals"] == res["finals"]
    t = O.relu_tables(Z, GA, Q, R)          # the returned points are the ones the claims are at
    assert v["claims"] == [O.mle_i32(Z, v["points"][0]), O.mle_i32(t["A"], v["points"][1]),
                           O.mle_i32(GA, v["points"][2]), O.mle_i32(t["GZ"], v["points"][3])]
    mproof = u32s(len(mg["r"]), 0, 2) + frs([mg["claim"]]) + frs([v for row in mg["msgs"] for v in row]) + frs(mg["finals"])
    vm = V.verify_relu_merge(H, logD, Q, R, res["point"], res["finals"], mproof)
    assert vm["point"] == mg["r"] and vm["claim"] == mg["finals"][0]
    assert H.state() == T.state()
    m = len(res["point"])
    for t in (0, m // 2, m - 1):
        bad = bytearray(proof)
        o = 12 + 128 + 128 * t + 32
        bad[o:o + 32] = ((int.from_bytes(bad[o:o + 32], "little") + 7) % P).to_bytes(32, "little")
        with pytest.raises(V.Rejected) as e:
            V.verify_relu(V.HostTranscript(seed=seed), bytes(bad), (logD, Q, R))
        assert e.value.where == t + 1
    bad = bytearray(proof)                   # sigma final changed: the six-statement identity fails
    bad[-32] ^= 0x01
    with pytest.raises(V.Rejected) as e:
        V.verify_relu(V.HostTranscript(seed=seed), bytes(bad), (logD, Q, R))
    assert e.value.where == -100
    bad = bytearray(proof)                   # a claim changed: round 1 fails
    bad[12] ^= 0x01
    with pytest.raises(V.Rejected) as e:
        V.verify_relu(V.HostTranscript(seed=seed), bytes(bad), (logD, Q, R))
    assert e.value.where == 1
    with pytest.raises(V.Rejected) as e:     # another statement shape
        V.verify_relu(V.HostTranscript(seed=seed), proof, (logD + 1, Q, R))
    assert e.value.where == -2
    with pytest.raises(ValueError):          # Q + R overflow guard
        V.verify_relu(V.HostTranscript(seed=seed), proof, (logD, 0xFFFFFFFF, 2))
    H2 = V.HostTranscript(seed=seed)         # the merge's weight final
    V.verify_relu(H2, proof, (logD, Q, R))
    badm = bytearray(mproof)
    badm[-32] ^= 0x01
    with pytest.raises(V.Rejected) as e:
        V.verify_relu_merge(H2, logD, Q, R, res["point"], res["finals"], bytes(badm))
    assert e.value.where in (-100, -101)


def test_window_verifier_on_oracle_window(V, oracle_lib):
    """D3d: a tiny FAC4DNN window proved by the oracle, verified family by family on forked host
    transcripts, joins replayed; a changed family proof is caught."""
    from oracle import drivers
    from synth import fcn
    shape = fcn.tiny_shape(steps=2, layers=3, width=8, batch=4, din=8, dout=4)
    trace = fcn.generate_trace(shape, x_bits=4, w_bits=4, y_bits=3)
    fams = fcn.assemble_families(shape, trace)
    o = drivers.fcn_prove(shape, fams, "vwin", merge_aux=True)
    results = []
    for f, r in zip(fams, o):
        r = dict(r)
        if hasattr(f, "A"):
            lN, l1, l2, l3 = r["logs"]
            r["proof"] = sc_proof(lN + l2, lN, 2, r)
        else:
            logD = int(f.Z.size).bit_length() - 1
            r["proof"] = relu_proof(logD, f.Q, f.R, r)
            mg = r["merge"]
            r["merge"] = dict(mg, proof=u32s(len(mg["r"]), 0, 2) + frs([mg["claim"]]) +
                              frs([v for row in mg["msgs"] for v in row]) + frs(mg["finals"]))
        results.append(r)
    out = V.verify_window(fs_seed("vwin"), fcn.fcn_header(shape), fams, results)
    assert [x["name"] for x in out] == [f.name for f in fams]
    for x, r, f in zip(out, o, fams):
        assert x["point"] == (r["r"] if "r" in r and "point" not in r else r["point"])
        assert x["finals"] == r["finals"]
        if hasattr(f, "A"):   # the matmul claim and its point are returned (open claims of the D3d window)
            assert (x["w"], x["u1"], x["u3"], x["claim"]) == (r["w"], r["u1"], r["u3"], r["claim"])
        else:
            assert x["claims"] == r["claims"] and x["merge_claim"] == r["merge"]["finals"][0]
    k = next(i for i, f in enumerate(fams) if hasattr(f, "A"))
    bad = dict(results[k])
    pb = bytearray(bad["proof"])
    pb[44] ^= 0x01
    bad["proof"] = bytes(pb)
    with pytest.raises(V.Rejected):
        V.verify_window(fs_seed("vwin"), fcn.fcn_header(shape), fams, results[:k] + [bad] + results[k + 1:])


def test_loss_grad_verifier(V, oracle_lib):
    """D24: the oracle's loss-gradient claims are accepted (end state = the oracle's), a false statement
    (one entry of G_Z changed) is rejected by the linear identity."""
    O = oracle_lib
    m = 7
    Z = uniform_range(43, 1, (1 << m,), -(1 << 20), 1 << 20)
    Y = uniform_range(43, 2, (1 << m,), -(1 << 20), 1 << 20)
    G = (Z.astype(np.int64) - Y).astype(np.int32)
    seed = fs_seed("vlg")
    T = O.Transcript(seed)
    res = O.loss_grad_prove(T, G, Z, Y)
    H = V.HostTranscript(seed=seed)
    assert V.verify_loss_grad(H, m, res["claims"]) == res["u"] and H.state() == T.state()
    G[3] -= 1
    bad = O.loss_grad_prove(O.Transcript(seed), G, Z, Y)
    with pytest.raises(V.Rejected) as e:
        V.verify_loss_grad(V.HostTranscript(seed=seed), m, bad["claims"])
    assert e.value.where == -100


def _merge_proof(mr):
    A, B = mr["A"], mr["B"]
    cA = sum(rh * c["c"] for rh, c in zip(mr["rho"], mr["claims_in"])) % P
    return (u32s(len(A["r"]), 0, 2) + frs([cA]) + frs([v for row in A["msgs"] for v in row]) + frs(A["finals"]) +
            u32s(len(B["r"]), 0, 2) + frs([A["finals"][1]]) + frs([v for row in B["msgs"] for v in row]) +
            frs(B["finals"]))


def _chained_results(o, fams, tensors, top=()):
    """The oracle's chained window in the device driver's result layout (proof bytes)."""
    res = dict(matmul={}, merges={}, relu={}, loss={}, rescale={}, window_state=o["window_state"])
    for f in top:
        r = dict(o["matmul"].get(f.name) or o["relu"][f.name])
        if hasattr(f, "Y"):
            res["loss"][f.name] = dict(u=r["u"], claims=r["claims"], state=r["state"])
        else:
            logD = int(f.Z.size).bit_length() - 1
            A, B = r["A"], r["B"]
            proof = (u32s(logD, f.Q, f.R) + frs(r["claims"]) +
                     u32s(len(A["r"]), 0, 2) + frs([(r["r"] * r["claims"][0] + r["claims"][1]) % P]) +
                     frs([v for row in A["msgs"] for v in row]) + frs(A["finals"]) +
                     u32s(len(B["r"]), len(B["r"]), 2) + frs([0]) + frs([v for row in B["msgs"] for v in row]) +
                     frs(B["finals"]))
            am = dict(r["aux_merge"])
            am["claims_in"] = [dict(c=A["finals"][1]), dict(c=B["finals"][0])]
            res["rescale"][f.name] = dict(proof=proof, aux_merge=dict(proof=_merge_proof(am)), state=r["state"])
    for f in fams:
        if hasattr(f, "A"):
            r = dict(o["matmul"][f.name])
            lN, l1, l2, l3 = r["logs"]
            r["proof"] = sc_proof(lN + l2, lN, 2, r)
            res["matmul"][f.name] = r
        else:
            r = dict(o["relu"][f.name])
            logD = int(f.Z.size).bit_length() - 1
            r["proof"] = relu_proof(logD, f.Q, f.R, r)
            mg = r["merge"]
            r["merge"] = dict(mg, proof=u32s(len(mg["r"]), 0, 2) + frs([mg["claim"]]) +
                              frs([v for row in mg["msgs"] for v in row]) + frs(mg["finals"]))
            res["relu"][f.name] = r
    for name, mr in o["merges"].items():
        res["merges"][name] = dict(mr, proof=_merge_proof(mr))
    return res


def _aux_mle(f, pt):
    """Brute-force MLE of the aux bit tensor aux[s][i][j] (s: Z / G_A words, j: bit, padded to B)."""
    from oracle import drivers  # noqa: F401
    import oracle as O
    QR = f.Q + f.R
    B = 1 << max(0, (QR - 1).bit_length())
    bits = []
    for w in (f.Z, f.GA):
        for v in np.asarray(w).reshape(-1):
            x = int(v) & 0xFFFFFFFF
            bits += [(x >> j) & 1 if j < QR else 0 for j in range(B)]
    return O.mle_fr(bits, pt)


def test_chained_window_verifier_on_oracle_window(V, oracle_lib):
    """N3 (D25): a tiny claim-chained window proved by the oracle; the host verifier accepts it and
    returns exactly one claim per committed tensor family plus the aux claim, each TRUE on the tensors
    (brute-force MLE); the zkReLU claims are bound to the merged claims; tampering anywhere is caught."""
    from oracle import drivers
    from synth import fcn
    O = oracle_lib
    O.set_threads(1)
    shape = fcn.tiny_shape(steps=2, layers=3, width=8, batch=4, din=8, dout=4)
    trace = fcn.generate_trace(shape, x_bits=4, w_bits=4, y_bits=3)
    fams = fcn.assemble_families(shape, trace)
    top = fcn.assemble_top_families(shape, trace, fams)
    tensors = fcn.plan_window(shape, trace, fams, top)
    o = drivers.fcn_prove_chained(shape, fams, tensors, "vchain", top=top)
    res = _chained_results(o, fams, tensors, top)
    hdr = fcn.fcn_header(shape)
    opened = V.verify_window_chained(fs_seed("vchain"), hdr, fams + top, tensors, res)
    assert opened == o["opened"]
    committed = [t for t in tensors if t.relu is None]
    relus = [f for f in fams if not hasattr(f, "A")]
    assert sorted(opened) == sorted([t.name for t in committed] + ["aux:" + f.name for f in relus + top[1:]])
    assert "Y" in opened and "Zout" not in opened and "Zp" not in opened      # the labels are data; Z^(L), Z' bound
    for t in committed:
        pt, val = opened[t.name]
        assert val == O.mle_i32(t.array.reshape(-1), pt), t.name
    for f in relus:
        pt, val = opened["aux:" + f.name]
        assert val == _aux_mle(f, pt)
    rs = top[1]                                  # the rescale's aux: the bits of Z^(L), [D][B]
    pt, val = opened["aux:" + rs.name]
    QR = rs.Q + rs.R
    bits = [((int(z) & 0xFFFFFFFF) >> j) & 1 if j < QR else 0 for z in rs.Z for j in range(32)]
    assert val == O.mle_fr(bits, pt)
    # a zkReLU proof whose claims are not the merged ones (a different Z claim) is rejected
    bad = dict(res, relu=dict(res["relu"]))
    f = relus[0]
    rr = dict(res["relu"][f.name])
    pb = bytearray(rr["proof"])
    pb[12] ^= 1
    rr["proof"] = bytes(pb)
    bad["relu"][f.name] = rr
    with pytest.raises(V.Rejected):
        V.verify_window_chained(fs_seed("vchain"), hdr, fams + top, tensors, bad)
    # a merge proof for other claims, and a missing merge
    name = next(iter(res["merges"]))
    bad = dict(res, merges=dict(res["merges"]))
    mb = bytearray(bad["merges"][name]["proof"])
    mb[20] ^= 1
    bad["merges"][name] = dict(bad["merges"][name], proof=bytes(mb))
    with pytest.raises(V.Rejected):
        V.verify_window_chained(fs_seed("vchain"), hdr, fams + top, tensors, bad)
    bad = dict(res, merges={k: v for k, v in res["merges"].items() if k != name})
    with pytest.raises(V.Rejected):
        V.verify_window_chained(fs_seed("vchain"), hdr, fams + top, tensors, bad)
