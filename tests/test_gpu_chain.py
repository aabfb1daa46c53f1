"""GPU parity of the claim-chained window (Protocol 1 lines 7-8; DESIGN.md
D25): chain.prove_window_chained against the oracle's drivers.fcn_prove_chained, bit-exact (D18), and
the library's host verifier (verify.verify_window_chained) on the GPU's bytes, with every opened claim
checked against the brute-force MLE of its tensor."""
import os

import numpy as np
import pytest
import torch

from synth.prng import DATA_SEED, fs_seed

pytestmark = pytest.mark.gpu
P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


@pytest.fixture(scope="module")
def ctx():
    from paper_2307_16273_b200 import build
    build.build(verbose=False)
    from paper_2307_16273_b200 import api
    return api.Context(0)


@pytest.fixture(scope="module")
def O():
    import oracle
    oracle.build()
    oracle.set_threads(len(os.sched_getaffinity(0)))
    return oracle


def _compare(g, o, fams, top=()):
    for f in top:
        if hasattr(f, "Y"):
            a, b = g["loss"][f.name], o["matmul"][f.name]
            assert a["u"] == b["u"] and a["claims"] == b["claims"] and a["state"] == b["state"], f.name
        else:
            a, b = g["rescale"][f.name], o["relu"][f.name]
            assert a["state"] == b["state"], f.name
            assert a["aux_merge"]["point"] == b["aux_merge"]["point"] and a["aux_merge"]["claim"] == b["aux_merge"]["claim"]
    for f in fams:
        if hasattr(f, "A"):
            a, b = g["matmul"][f.name], o["matmul"][f.name]
            assert (a["w"], a["u1"], a["u3"], a["claim"]) == (b["w"], b["u1"], b["u3"], b["claim"]), f.name
            assert a["msgs"] == b["msgs"] and a["finals"] == b["finals"] and a["state"] == b["state"], f.name
    assert set(g["merges"]) == set(o["merges"])
    for name, b in o["merges"].items():
        a = g["merges"][name]
        assert a["A"]["msgs"] == b["A"]["msgs"] and a["A"]["finals"] == b["A"]["finals"], name
        assert a["B"]["msgs"] == b["B"]["msgs"] and a["B"]["finals"] == b["B"]["finals"], name
        assert a["point"] == b["point"] and a["claim"] == b["claim"] and a["state"] == b["state"], name


def _run(ctx, O, shape, seed_name, streams, x_bits=11, w_bits=12, y_bits=10, full_oracle=True):
    from paper_2307_16273_b200 import api, chain, verify
    from oracle import drivers
    from synth import fcn
    trace = fcn.generate_trace(shape, seed=DATA_SEED, x_bits=x_bits, w_bits=w_bits, y_bits=y_bits)
    fams = fcn.assemble_families(shape, trace)
    top = fcn.assemble_top_families(shape, trace, fams)
    tensors = fcn.plan_window(shape, trace, fams, top)
    dfams, dts = chain.upload_plan(fams, tensors, top=top)
    relu_ctx = api.Context(0, torch.cuda.Stream()) if streams else None
    mm = [api.Context(0, torch.cuda.Stream()) for _ in range(streams)]
    # with streams: the bench's stage-3 layout (the rescale and the late claim merges beside the zkReLU, on
    # budgeted streams)
    rs = api.Context(0, torch.cuda.Stream()) if streams else None
    late = [api.Context(0, torch.cuda.Stream()) for _ in range(2 * streams)]
    for c in ([rs] if rs else []) + late:
        c.set_sm_budget(12)
        c.set_persistent(False)
    g = chain.prove_window_chained(ctx, fs_seed(seed_name), fcn.fcn_header(shape), dfams, dts, relu_ctx=relu_ctx,
                                   mm_ctxs=mm, rescale_ctx=rs, late_ctxs=late or None)
    opened = verify.verify_window_chained(fs_seed(seed_name), fcn.fcn_header(shape), fams + top, tensors, g)
    return fams, top, tensors, g, opened


def test_chained_window_tiny_vs_oracle(ctx, O):
    """A tiny window (2 steps, 3 layers): every family, merge and the chained zkReLU bit-exact against
    the oracle; the opened claims equal the oracle's and are true on the tensors."""
    from oracle import drivers
    from synth import fcn
    shape = fcn.tiny_shape(steps=2, layers=3, width=8, batch=4, din=8, dout=4)
    for streams in (0, 2):
        fams, top, tensors, g, opened = _run(ctx, O, shape, "chain-tiny", streams, x_bits=4, w_bits=4, y_bits=3)
        o = drivers.fcn_prove_chained(shape, fams, tensors, "chain-tiny", top=top)
        _compare(g, o, fams, top)
        for f in fams:
            if not hasattr(f, "A"):
                a, b = g["relu"][f.name], o["relu"][f.name]
                assert a["claims"] == b["claims"] and a["msgs"] == b["msgs"] and a["finals"] == b["finals"]
                assert a["merge"]["msgs"] == b["merge"]["msgs"] and a["state"] == b["state"]
        assert g["window_state"] == o["window_state"]
        assert opened == o["opened"]


@pytest.mark.parametrize("layers,width", [(4, 64), (3, 256)])
def test_chained_window_mid_vs_oracle(ctx, O, layers, width):
    """Wider windows (several tiles per kernel, padded stacks: 3 ReLU layers x 2 steps = 6 -> 8 slots)."""
    from oracle import drivers
    from synth import fcn
    shape = fcn.tiny_shape(steps=2, layers=layers, width=width, batch=16, din=width * 2, dout=16)
    fams, top, tensors, g, opened = _run(ctx, O, shape, f"chain-{layers}-{width}", 2)
    o = drivers.fcn_prove_chained(shape, fams, tensors, f"chain-{layers}-{width}", top=top)
    _compare(g, o, fams, top)
    for f in fams:
        if not hasattr(f, "A"):
            assert g["relu"][f.name]["msgs"] == o["relu"][f.name]["msgs"]
    assert g["window_state"] == o["window_state"] and opened == o["opened"]


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_chained_window_full_size(ctx, O, cfg):
    """C3 and C4 (the bench workload) chained, in the bench's stream configuration: every matmul family
    and every claim merge bit-exact against the oracle; the chained zkReLU accepted by the oracle's
    verifier at the merged points (claims = brute-force MLEs there); the library's host verifier accepts
    the window; every opened committed claim equals the brute-force MLE of its stack."""
    from oracle import drivers
    from synth import fcn
    shape = fcn.C4_SHAPE if cfg == "C4" else fcn.C3_SHAPE
    fams, top, tensors, g, opened = _run(ctx, O, shape, f"{cfg}-chained", 2)
    # the oracle: stages 1 and 2 in full (the driver's pieces), then the zkReLU through the oracle's verifier
    # at the merged points (the dense oracle zkReLU of 2^28 entries is out of reach), the rescale in full
    import oracle as Ol
    W = Ol.Transcript(fs_seed(f"{cfg}-chained"))
    W.absorb("fcn/chdr", fcn.fcn_header(shape))
    mms = [f for f in fams if hasattr(f, "A")]
    loss, resc = top
    kids = []
    for f in mms + [loss]:
        W.absorb("fcn/fam", f.name.encode())
        kids.append(Ol.Transcript(W.challenges("fcn/fork", 1)[0].to_bytes(32, "little")))
    om = {}
    for f, T in zip(mms, kids):
        r = Ol.matmul_prove(T, f.A, f.B, f.transA, f.transB)
        r["state"] = T.state()
        om[f.name] = r
    ol = Ol.loss_grad_prove(kids[-1], loss.GZ, loss.Zp, loss.Y)
    ol["state"] = kids[-1].state()
    _compare(dict(matmul=g["matmul"], merges={}, loss=g["loss"]), dict(matmul=dict(om, **{loss.name: ol}), merges={}),
             fams, [loss])
    for T in kids:
        W.absorb("fcn/join", T.state())
    claims = {t.name: [] for t in tensors}
    for f in mms:
        for role, ref, v, u, c in drivers._matmul_family_claims(f, om[f.name]):
            claims[ref.tensor].append(dict(map=list(ref.map), u=list(u), v=list(v), c=c))
    for role, ref, v, u, c in drivers._loss_family_claims(loss, ol):
        claims[ref.tensor].append(dict(map=list(ref.map), u=list(u), v=list(v), c=c))
    merged = [t for t in tensors if claims[t.name] and not drivers._is_whole(t, claims[t.name])]
    assert sorted(t.name for t in merged) == sorted(g["merges"])
    # D25 order: the merges stage 3 is bound to, joined; stage 3's forks; the other merges' forks
    st3 = [f for f in fams if not hasattr(f, "A")] + [resc]
    bound = {f.tensors[k] for f in st3 if f is not resc for k in ("Z", "A", "GA", "GZ")} | \
        {resc.tensors["Z"], resc.tensors["Zp"]}
    merged_a = [t for t in merged if t.name in bound]
    merged_b = [t for t in merged if t.name not in bound]
    one = {}
    for t in tensors:
        if claims[t.name] and t not in merged:
            one[t.name] = (claims[t.name][0]["v"] + claims[t.name][0]["u"], claims[t.name][0]["c"])

    def check_merges(ts, ks):
        for t, T in zip(ts, ks):
            r = Ol.claim_merge_prove(T, drivers._tensor_values(t, fams + top), claims[t.name])
            a = g["merges"][t.name]
            assert a["A"]["msgs"] == r["A"]["msgs"] and a["B"]["msgs"] == r["B"]["msgs"], t.name
            assert a["point"] == r["point"] and a["claim"] == r["claim"] and a["state"] == T.state(), t.name
            one[t.name] = (r["point"], r["claim"])

    mk = []
    for t in merged_a:
        W.absorb("fcn/tfam", t.name.encode())
        mk.append(Ol.Transcript(W.challenges("fcn/fork", 1)[0].to_bytes(32, "little")))
    check_merges(merged_a, mk)
    for T in mk:
        W.absorb("fcn/join", T.state())
    forks3 = []
    for f in st3:                      # D25 stage 3: every fork first, then the proofs, then the joins
        W.absorb("fcn/fam", f.name.encode())
        forks3.append(Ol.Transcript(W.challenges("fcn/fork", 1)[0].to_bytes(32, "little")))
    mkb = []
    for t in merged_b:
        W.absorb("fcn/tfam", t.name.encode())
        mkb.append(Ol.Transcript(W.challenges("fcn/fork", 1)[0].to_bytes(32, "little")))
    check_merges(merged_b, mkb)
    for f, T in zip(st3, forks3):
        if f is resc:
            r = Ol.rescale_prove(T, f.Z, f.Q, f.R, [one[f.tensors["Z"]][0], one[f.tensors["Zp"]][0]])
            assert r["claims"] == [one[f.tensors["Z"]][1], one[f.tensors["Zp"]][1]]
            logB = Ol.relu_logB(f.Q, f.R)
            bits = ((f.Z.astype(np.int64).reshape(-1, 1) & 0xFFFFFFFF) >> np.arange(1 << logB)) & 1
            bits[:, f.Q + f.R:] = 0
            am = Ol.claim_merge_prove(T, np.ascontiguousarray(bits.astype(np.int32).reshape(1, -1)),
                                      [dict(map=[0], u=[], v=r["A"]["r"], c=r["A"]["finals"][1]),
                                       dict(map=[0], u=[], v=r["B"]["r"], c=r["B"]["finals"][0])])
            ga = g["rescale"][f.name]
            assert ga["aux_merge"]["point"] == am["point"] and ga["aux_merge"]["claim"] == am["claim"]
            assert ga["state"] == T.state()
            continue
        gr = g["relu"][f.name]
        pts = [one[f.tensors[k]][0] for k in ("Z", "A", "GA", "GZ")]
        assert Ol.relu_verify(T, f.Z, f.GA, f.Q, f.R, gr["claims"], gr["msgs"], gr["finals"], points=pts) == 0
        assert gr["claims"] == [one[f.tensors[k]][1] for k in ("Z", "A", "GA", "GZ")]
        rho = T.challenges("relu/merge", 1)[0]
        f0, f1, f2 = gr["finals"]
        assert gr["merge"]["claim"] == (f0 + rho * f1 + rho * rho * f2) % P
        assert Ol.sumcheck_verify(T, len(gr["merge"]["r"]), 0, 2, [], gr["merge"]["claim"], gr["merge"]["msgs"],
                                  gr["merge"]["finals"]) == 0
        assert gr["state"] == T.state()
    for T in forks3 + mkb:
        W.absorb("fcn/join", T.state())
    assert g["window_state"] == W.state()
    for t in tensors:
        if t.relu is None and t.name in opened:
            pt, val = opened[t.name]
            assert val == Ol.mle_i32(np.ascontiguousarray(t.array).reshape(-1), pt), t.name


@pytest.mark.parametrize("logD,Q,R", [(5, 16, 16), (12, 16, 16), (14, 16, 16), (16, 16, 16), (17, 16, 16), (10, 8, 8)])
def test_rescale_vs_oracle(ctx, O, logD, Q, R):
    """zk_rescale_prove_dev (D26) against the oracle at given points: claims, both sumchecks' messages and
    finals bit-exact (the larger sizes through the factored round kernels with an Fr and an int32 table),
    and the library's host verifier accepts and ends in the prover's state."""
    import random
    from paper_2307_16273_b200 import api, verify
    from synth.prng import uniform_range
    rng = random.Random(logD)
    half = 1 << (Q + R - 1)
    Z = uniform_range(46, logD, (1 << logD,), -half, half)
    pts = [[rng.randrange(P) for _ in range(logD)] for _ in range(2)]
    seed = fs_seed(f"rescale-{logD}-{Q}")
    o = O.rescale_prove(O.Transcript(seed), Z, Q, R, pts)
    tr = api.Transcript(ctx, seed)
    d_pts = torch.frombuffer(bytearray(b"".join(int(x).to_bytes(32, "little") for u in pts for x in u)),
                             dtype=torch.uint8).cuda()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = api.rescale_prove_dev(ctx, tr, torch.from_numpy(Z).cuda(), Q, R, d_pts, flag)
    g = api.parse_rescale_out(out.cpu().numpy().tobytes(), logD, Q, R)
    assert int(flag.item()) == 0
    assert g["claims"] == o["claims"]
    assert g["A"]["msgs"] == o["A"]["msgs"] and g["A"]["finals"] == o["A"]["finals"] and g["A"]["r"] == o["A"]["r"]
    assert g["B"]["msgs"] == o["B"]["msgs"] and g["B"]["finals"] == o["B"]["finals"] and g["B"]["r"] == o["B"]["r"]
    H = verify.HostTranscript(seed=seed)
    v = verify.verify_rescale(H, g["proof"], (logD, Q, R), pts)
    assert v["claims"] == o["claims"] and v["aux"] == [o["A"]["finals"][1], o["B"]["finals"][0]]
    assert H.state() == tr.state()


@pytest.mark.parametrize("n,lr,lc,source,K", [(0, 14, 5, "bits", 2), (0, 16, 5, "bits", 2), (0, 16, 5, "plain", 2),
                                              (3, 4, 6, "plain", 3), (7, 6, 10, "plain", 2), (2, 8, 8, "plain", 5)])
def test_claim_merge_vs_oracle(ctx, O, n, lr, lc, source, K):
    """zk_claim_merge_dev (D25) against the oracle: single-slice stacks of bit columns (the rescale's aux)
    and plain stacks with partial views, bit-exact; the host verifier accepts."""
    import random
    from paper_2307_16273_b200 import api, verify
    from synth.prng import uniform_range
    rng = random.Random(n * 100 + lr + lc + K)
    d = lr + lc
    N = 1 << n
    if source == "bits":
        Zw = uniform_range(47, lr, (1 << lr,), -(1 << 31), 1 << 31)
        X = ((Zw.astype(np.int64).reshape(-1, 1) & 0xFFFFFFFF) >> np.arange(1 << lc)) & 1
        X = np.ascontiguousarray(X.astype(np.int32).reshape(1, -1))
    else:
        X = uniform_range(47, n + d, (N, 1 << d), -(1 << 31), 1 << 31)
    claims = []
    for k in range(K):
        nk = rng.randrange(0, n + 1) if n else 0
        pick = rng.sample(range(N), min(1 << nk, N))
        mp = pick + [-1] * ((1 << nk) - len(pick))
        rng.shuffle(mp)
        u = [rng.randrange(P) for _ in range(nk)]
        v = [rng.randrange(P) for _ in range(d)]
        c = 0
        for j, i in enumerate(mp):              # the honest claim X_k~(v, u) = sum_j beta(u, j) X_map[j]~(v)
            if i >= 0:
                b = 1
                for t, x in enumerate(u):
                    b = b * (x if (j >> t) & 1 else 1 - x) % P
                c = (c + b * O.mle_i32(X[i], v)) % P
        claims.append(dict(map=mp, u=u, v=v, c=c))
    seed = fs_seed(f"cm-{n}-{lr}-{lc}-{K}")
    o = O.claim_merge_prove(O.Transcript(seed), X, claims)
    tr = api.Transcript(ctx, seed)
    pts = b"".join(int(x).to_bytes(32, "little") for c in claims for x in c["v"] + c["u"])
    cls = b"".join(int(c["c"]).to_bytes(32, "little") for c in claims)
    dp = torch.frombuffer(bytearray(pts), dtype=torch.uint8).cuda()
    dc = torch.frombuffer(bytearray(cls), dtype=torch.uint8).cuda()
    if source == "bits":
        out = api.claim_merge_dev(ctx, tr, torch.from_numpy(Zw).cuda(), 0, lr, lc, [c["map"] for c in claims], dp, dc,
                                  source="bits", R=32)
    else:
        out = api.claim_merge_dev(ctx, tr, torch.from_numpy(X).cuda(), n, lr, lc, [c["map"] for c in claims], dp, dc)
    g = api.parse_claim_merge_out(out.cpu().numpy().tobytes(), n, K, d)
    assert g["A"]["msgs"] == o["A"]["msgs"] and g["A"]["finals"] == o["A"]["finals"]
    assert g["B"]["msgs"] == o["B"]["msgs"] and g["B"]["finals"] == o["B"]["finals"]
    assert g["point"] == o["point"] and g["claim"] == o["claim"]
    H = verify.HostTranscript(seed=seed)
    assert verify.verify_claim_merge(H, n, d, claims, g["proof"]) == (o["point"], o["claim"])
    assert H.state() == tr.state()
