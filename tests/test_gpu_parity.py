"""GPU parity: every CUDA entry point against the CPU oracle on the same seeded inputs.

Bit-exact (D18): transcripts, messages, claims, points and finals must be
identical integers.  Sizes span several tiles/blocks and ragged grid tails;
full-size configurations are checked by the oracle verifier (round identities,
final identities, finals against brute-force MLE of the inputs).
"""
import random

import numpy as np
import pytest
import torch

from synth.prng import fs_seed, uniform_range

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
    return oracle


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ---------------------------------------------------------------- Fr arithmetic
def test_fr_ops_vs_python_ints(ctx):
    from paper_2307_16273_b200 import api
    rng = random.Random(1)
    edges = [0, 1, 2, P - 1, P - 2, (1 << 256) % P, (1 << 255) % P, (1 << 32) - 1, 1 << 32, (1 << 64) - 1,
             P >> 1, (P >> 1) + 1]
    a = edges + [rng.randrange(P) for _ in range(4000)]
    b = [rng.choice(edges) for _ in edges] + [rng.randrange(P) for _ in range(4000)]
    b = b[:len(a)]
    ta, tb = api.fr_table_from_ints(ctx, a), api.fr_table_from_ints(ctx, b)
    assert api.fr_table_to_ints(ctx, ta) == a
    for op, f in [("add", lambda x, y: (x + y) % P), ("sub", lambda x, y: (x - y) % P),
                  ("mul", lambda x, y: x * y % P)]:
        got = api.fr_table_to_ints(ctx, api.diag_fr_op(ctx, op, ta, tb))
        assert got == [f(x, y) for x, y in zip(a, b)], op
    got = api.fr_table_to_ints(ctx, api.diag_fr_op(ctx, "sqr", ta))
    assert got == [x * x % P for x in a]
    got = api.fr_table_to_ints(ctx, api.diag_fr_op(ctx, "neg", ta))
    assert got == [(-x) % P for x in a]
    small = api.fr_table_from_ints(ctx, a[1:200])
    got = api.fr_table_to_ints(ctx, api.diag_fr_op(ctx, "inv", small))
    assert got == [pow(x, P - 2, P) for x in a[1:200]]
    got = api.fr_table_to_ints(ctx, api.diag_fr_op(ctx, "inv_bgcd", small))   # the u^-1 kernels' inversion
    assert got == [pow(x, P - 2, P) for x in a[1:200]]


def test_noncanonical_rejected(ctx):
    from paper_2307_16273_b200 import api
    from paper_2307_16273_b200._lib import ZkError
    raw = torch.frombuffer(bytearray(P.to_bytes(32, "little")), dtype=torch.uint8).reshape(1, 32).cuda()
    with pytest.raises(ZkError):
        api.fr_table_from_canonical(ctx, raw)
    import ctypes
    from paper_2307_16273_b200._lib import lib
    out = api.fr_empty(2, "cuda")
    st = lib().zk_eq_table(ctx.h, ctypes.create_string_buffer(P.to_bytes(32, "little"), 32), 1, None, out.data_ptr())
    assert st == -3    # ZK_ERR_NONCANONICAL


# ---------------------------------------------------------------- transcript (D3)
def test_transcript_vs_oracle(ctx, O):
    from paper_2307_16273_b200 import api
    seed = fs_seed("gpu-transcript")
    g, o = api.Transcript(ctx, seed), O.Transcript(seed)
    rng = random.Random(2)
    for step in range(40):
        if step % 3 == 0:
            msg = bytes(rng.randrange(256) for _ in range(rng.choice([0, 1, 12, 55, 56, 64, 119, 300, 1000])))
            g.absorb("t/abs", msg)
            o.absorb("t/abs", msg)
        else:
            n = rng.choice([1, 2, 5, 33, 300])
            assert g.challenges("t/ch", n) == o.challenges("t/ch", n)
    assert g.state() == o.state()


# ---------------------------------------------------------------- tables (rows a1, a2)
def test_embed(ctx):
    from paper_2307_16273_b200 import api
    v = uniform_range(3, 3, (5000,), -(1 << 31), 1 << 31)
    v[:4] = [0, -1, (1 << 31) - 1, -(1 << 31)]
    got = api.fr_table_to_ints(ctx, api.embed_i32(ctx, dev(v)))
    assert got == [int(x) % P for x in v]


@pytest.mark.parametrize("k", [0, 1, 3, 10, 11, 14])
def test_eq_table(ctx, O, k):
    from paper_2307_16273_b200 import api
    rng = random.Random(k)
    u = [rng.randrange(P) for _ in range(k)]
    assert api.fr_table_to_ints(ctx, api.eq_table(ctx, u)) == O.eq_table(u)
    s = rng.randrange(P)
    assert api.fr_table_to_ints(ctx, api.eq_table(ctx, u, scale=s)) == [x * s % P for x in O.eq_table(u)]


@pytest.mark.parametrize("m", [1, 5, 12, 13, 17])
def test_mle(ctx, O, m):
    from paper_2307_16273_b200 import api
    rng = random.Random(m)
    u = [rng.randrange(P) for _ in range(m)]
    t = uniform_range(4, m, (1 << m,), -(1 << 31), 1 << 31)
    assert api.mle_eval_i32(ctx, dev(t), u) == O.mle_i32(t, u)
    tf = api.embed_i32(ctx, dev(t))
    assert api.mle_eval_fr(ctx, tf, u) == O.mle_i32(t, u)


# ---------------------------------------------------------------- product sumcheck (rows a4-a6)
SC_CASES = [(1, 0, 1), (1, 1, 2), (2, 2, 3), (3, 0, 2), (6, 6, 2), (8, 3, 3), (10, 10, 1), (11, 11, 2),
            (12, 12, 2), (13, 12, 2), (14, 14, 3), (16, 5, 2), (17, 17, 2)]


@pytest.mark.parametrize("m,n_eq,K", SC_CASES)
def test_sumcheck_vs_oracle(ctx, O, m, n_eq, K):
    from paper_2307_16273_b200 import api
    rng = random.Random(m * 1000 + n_eq * 10 + K)
    tabs = [uniform_range(7, 100 * m + k, (1 << m,), -(1 << 15), 1 << 15) for k in range(K)]
    w = [rng.randrange(P) for _ in range(n_eq)]
    seed = fs_seed(f"sc-{m}-{n_eq}-{K}")
    give_claim = (m % 2 == 0)
    ot = [[int(v) % P for v in t] for t in tabs]
    o = O.sumcheck_prove(O.Transcript(seed), m, n_eq, ot, w, None)
    claim = o["claim"] if give_claim else None
    # mix int32 and Fr inputs
    gt = [dev(t) if k % 2 == 0 else api.embed_i32(ctx, dev(t)) for k, t in enumerate(tabs)]
    tr = api.Transcript(ctx, seed)
    g = api.sumcheck_prove(ctx, tr, m, n_eq, gt, w, claim)
    assert g["claim"] == o["claim"]
    assert g["msgs"] == o["msgs"]
    assert g["r"] == o["r"]
    assert g["finals"] == o["finals"]
    ot2 = O.Transcript(seed)
    O.sumcheck_prove(ot2, m, n_eq, ot, w, claim)
    assert tr.state() == ot2.state()


# ---------------------------------------------------------------- matmul (row a3)
MM_CASES = [(0, 5, 6, 6, False, False), (2, 3, 4, 2, False, False), (3, 4, 5, 3, True, False),
            (2, 6, 7, 5, False, True), (1, 6, 6, 10, True, True), (4, 2, 9, 12, False, True), (3, 10, 6, 4, True, False),
            # the row-streaming column sums (k_colsum_rows: 512 / 1024 columns, CTA ranges straddling instances)
            (4, 10, 9, 0, False, False), (3, 0, 10, 11, False, True)]


@pytest.mark.parametrize("lN,l1,l2,l3,ta,tb", MM_CASES)
def test_matmul_vs_oracle(ctx, O, lN, l1, l2, l3, ta, tb):
    from paper_2307_16273_b200 import api
    N, D1, D2, D3 = 1 << lN, 1 << l1, 1 << l2, 1 << l3
    A = uniform_range(8, 1 + lN, (N, D2, D1) if ta else (N, D1, D2), -(1 << 15), 1 << 15)
    B = uniform_range(8, 2 + l3, (N, D3, D2) if tb else (N, D2, D3), -(1 << 15), 1 << 15)
    seed = fs_seed(f"mm-{lN}-{l1}-{l2}-{l3}")
    o = O.matmul_prove(O.Transcript(seed), A, B, ta, tb)
    tr = api.Transcript(ctx, seed)
    red = api.matmul_reduce(ctx, tr, dev(A), dev(B), ta, tb)
    assert (red["w"], red["u1"], red["u3"]) == (o["w"], o["u1"], o["u3"])
    assert api.fr_table_to_ints(ctx, red["At"]) == o["At"]
    assert api.fr_table_to_ints(ctx, red["Bt"]) == o["Bt"]
    assert red["claim"] == o["claim"]
    g = api.sumcheck_prove(ctx, tr, lN + l2, lN, [red["At"], red["Bt"]], red["w"], red["claim"])
    assert g["msgs"] == o["msgs"] and g["finals"] == o["finals"] and g["r"] == o["r"]


def test_c1_golden(ctx):
    """C1 (BASELINE configs[0]) against the frozen oracle transcript (tests/golden, written from oracle/ only)."""
    import json
    import os
    from oracle import drivers
    from paper_2307_16273_b200 import api
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c1_transcript.json")))
    A, B = drivers.c1_inputs()
    tr = api.Transcript(ctx, fs_seed("C1"))
    red = api.matmul_reduce(ctx, tr, dev(A), dev(B))
    g = api.sumcheck_prove(ctx, tr, 6, 0, [red["At"], red["Bt"]], red["w"], red["claim"])
    assert hex(red["claim"]) == gold["claim"]
    assert [[hex(v) for v in row] for row in g["msgs"]] == gold["msgs"]
    assert [hex(v) for v in g["finals"]] == gold["finals"]
    assert tr.state().hex() == gold["final_state"]


# ---------------------------------------------------------------- zkReLU (rows a7, a8)
def test_relu_tables_vs_oracle(ctx, O):
    from paper_2307_16273_b200 import api
    for (Q, R) in [(4, 2), (16, 16), (8, 8)]:
        half = 1 << (Q + R - 1)
        Z = uniform_range(9, Q, (4096,), -half, half)
        GA = uniform_range(9, Q + 1, (4096,), -half, half)
        o = O.relu_tables(Z, GA, Q, R)
        g = api.relu_tables(ctx, dev(Z), dev(GA), Q, R)
        for k in ("A", "GZ", "Zp", "GAp", "RZ", "RGA", "sign"):
            assert np.array_equal(g[k].cpu().numpy(), o[k]), (Q, R, k)
    from paper_2307_16273_b200._lib import ZkError
    with pytest.raises(ZkError):
        api.relu_tables(ctx, dev(np.array([32, 0], np.int32)), dev(np.array([0, 0], np.int32)), 4, 2)


# logD >= 12 with B >= 8 runs the tensor-core bit sums (gram.cu): (16,16,12) gives most CTAs one or two
# K steps, (16,16,17) crosses a 2^16-entry row inside CTAs, (4,4,12) and (8,8,14) have B = 8 and 16.
RELU_CASES = [(4, 2, 1), (4, 2, 3), (4, 2, 6), (4, 4, 5), (16, 16, 2), (16, 16, 6), (8, 8, 9), (16, 16, 11),
              (12, 4, 8), (16, 16, 13), (16, 16, 12), (4, 4, 12), (8, 8, 14), (12, 4, 15), (16, 16, 17)]


@pytest.mark.parametrize("Q,R,logD", RELU_CASES)
def test_relu_vs_oracle(ctx, O, Q, R, logD):
    from paper_2307_16273_b200 import api
    half = 1 << (Q + R - 1)
    Z = uniform_range(10, 7 * logD + Q, (1 << logD,), -half, half)
    GA = uniform_range(10, 7 * logD + R + 100, (1 << logD,), -half, half)
    Z[:2] = [-1, half - 1]          # D10/D11 edges
    seed = fs_seed(f"relu-{Q}-{R}-{logD}")
    o = O.relu_prove(O.Transcript(seed), Z, GA, Q, R)
    tr = api.Transcript(ctx, seed)
    g = api.relu_prove(ctx, tr, dev(Z), dev(GA), Q, R)
    assert g["claims"] == o["claims"]
    for t, (gm, om) in enumerate(zip(g["msgs"], o["msgs"])):
        assert gm == om, f"round {t}"
    assert g["point"] == o["point"]
    assert g["finals"] == o["finals"]


def test_relu_range_error(ctx):
    from paper_2307_16273_b200 import api
    from paper_2307_16273_b200._lib import ZkError
    Z = np.zeros(16, np.int32)
    Z[3] = 40
    with pytest.raises(ZkError):
        api.relu_prove(ctx, api.Transcript(ctx, bytes(32)), dev(Z), dev(np.zeros(16, np.int32)), 4, 2)


@pytest.mark.parametrize("env", [{"ZKDL_IPERSIST_LOG": "-1"}, {"ZKDL_IPERSIST_LOG": "5"}, {"ZKDL_IPERSIST_LOG": "30"},
                                 {"ZKDL_IROUND_V": "0"}])
@pytest.mark.parametrize("logD", [12, 17])
def test_relu_round_paths_vs_oracle(ctx, O, logD, env, monkeypatch):
    """Every i-round path gives the oracle's transcript: per-round factored launches only, a switch to
    the persistent kernel mid-way, persistent from round 1, and the unfactored A/B kernel."""
    from paper_2307_16273_b200 import api
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    Z = uniform_range(11, 3 * logD, (1 << logD,), -(1 << 31), 1 << 31)
    GA = uniform_range(11, 3 * logD + 1, (1 << logD,), -(1 << 31), 1 << 31)
    seed = fs_seed(f"relu-paths-{logD}")
    o = O.relu_prove(O.Transcript(seed), Z, GA, 16, 16)
    g = api.relu_prove(ctx, api.Transcript(ctx, seed), dev(Z), dev(GA), 16, 16)
    assert g["msgs"] == o["msgs"] and g["finals"] == o["finals"]


def test_c2_full_vs_oracle(ctx, O):
    """C2 (BASELINE configs[1]) at full size: 64 x 1024 entries, Q = R = 16, bit-exact against the dense oracle."""
    from oracle import drivers
    from paper_2307_16273_b200 import api
    Z, GA = drivers.c2_inputs()
    o = drivers.c2_prove()
    tr = api.Transcript(ctx, fs_seed("C2"))
    g = api.relu_prove(ctx, tr, dev(Z), dev(GA), 16, 16)
    assert g["claims"] == o["claims"] and g["msgs"] == o["msgs"] and g["finals"] == o["finals"]
    assert tr.state() == o["state"]


# ---------------------------------------------------------------- C5 single sumcheck
@pytest.mark.parametrize("m", [12, 17, 19])
def test_c5_vs_oracle(ctx, O, m):
    from oracle import drivers
    from paper_2307_16273_b200 import api
    A, B = drivers.c5_inputs(m)
    o = drivers.c5_prove(m)
    tr = api.Transcript(ctx, fs_seed(f"C5-m{m}"))
    tr.absorb("c5/hdr", m.to_bytes(4, "little"))
    w = tr.challenges("c5/w", m)
    g = api.sumcheck_prove(ctx, tr, m, m, [dev(A), dev(B)], w, None)
    assert g["claim"] == o["claim"] and g["msgs"] == o["msgs"] and g["finals"] == o["finals"]
    assert tr.state() == o["state"]


@pytest.mark.parametrize("m,switch", [(17, None), (18, None), (18, 40), (18, 17)])
def test_int_round0_extreme_values_vs_oracle(ctx, O, m, switch):
    """The integer round 0 (k_sc_round0_int) and the int32 fold of round 1 at the extremes of int32:
    P(inf) = (a1 - a0)(b1 - b0) reaches (2^32 - 1)^2 > 2^63, P(0), P(1) reach 2^62; m = 17 hands round 1
    to the persistent tail (the int32 tables are embedded first); through the shard session, switch = 40
    exports before round 0, switch = m - 1 exports the int32 fold after the integer round 0."""
    from paper_2307_16273_b200 import api, shard
    rng = random.Random(77 + m)
    A = uniform_range(14, m, (1 << m,), -(1 << 31), 1 << 31)
    B = uniform_range(14, m + 50, (1 << m,), -(1 << 31), 1 << 31)
    lo, hi = np.int32(-(1 << 31)), np.int32((1 << 31) - 1)
    A[0::4], A[1::4], B[0::4], B[1::4] = lo, hi, hi, lo        # maximal |a1 - a0|, |b1 - b0|, opposite signs
    A[2::8], B[2::8] = lo, lo                                    # (-2^31)^2 = 2^62
    w = [rng.randrange(P) for _ in range(m)]
    seed = fs_seed(f"int0-{m}")
    o = O.sumcheck_prove(O.Transcript(seed), m, m, [[int(v) % P for v in t] for t in (A, B)], w, None)
    if switch is None:
        g = api.sumcheck_prove(ctx, api.Transcript(ctx, seed), m, m, [dev(A), dev(B)], w, None)
        assert g["claim"] == o["claim"] and g["msgs"] == o["msgs"] and g["finals"] == o["finals"]
    else:
        sess = shard.ShardSession(ctx, api.Transcript(ctx, seed), m, m, [dev(A), dev(B)], w, 0, 1)
        r = shard.prove_virtual([sess], switch_log=switch)
        assert r[0]["msgs"] == o["msgs"] and r[0]["finals"] == o["finals"]
        sess.close()


# ---------------------------------------------------------------- FCN family driver (row a9)
def test_fcn_tiny_vs_oracle(ctx, O):
    from oracle import drivers
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    shape = fcn.tiny_shape(steps=2, layers=3, width=8, batch=4, din=8, dout=4)
    trace = fcn.generate_trace(shape, x_bits=4, w_bits=4, y_bits=3)
    fams = fcn.assemble_families(shape, trace)
    o = drivers.fcn_prove(shape, fams, "tiny")
    g = dfcn.prove_window(ctx, fs_seed("tiny"), fcn.fcn_header(shape), dfcn.upload_families(fams))
    assert len(g) == len(o)
    for gr, orr in zip(g, o):
        assert gr["msgs"] == orr["msgs"], gr["name"]
        assert gr["finals"] == orr["finals"], gr["name"]
        assert gr["state"] == orr["state"], gr["name"]
    assert g[-1]["window_state"] == o[-1]["window_state"]          # D3d joins
    # end-to-end entry (host tensors, per-family uploads overlapped with proofs) with the zkReLU
    # family on a second stream: same bytes
    import torch
    from paper_2307_16273_b200 import api
    relu_ctx = api.Context(0, torch.cuda.Stream())
    host = dfcn.upload_families(fams, device="cpu")
    h = dfcn.prove_window_from_host(ctx, fs_seed("tiny"), fcn.fcn_header(shape), host, relu_ctx=relu_ctx)
    assert [r["proof"] for r in h] == [r["proof"] for r in g]
    hh = dfcn.prove_windows_from_host(ctx, [(fs_seed("tiny"), fcn.fcn_header(shape), host)] * 3, relu_ctx=relu_ctx)
    assert all([r["proof"] for r in w] == [r["proof"] for r in g] for w in hh)
    assert [r["state"] for r in h] == [r["state"] for r in g]
    assert h[-1]["window_state"] == g[-1]["window_state"]
    g2 = dfcn.prove_window(ctx, fs_seed("tiny"), fcn.fcn_header(shape), dfcn.upload_families(fams), relu_ctx=relu_ctx)
    assert [r["proof"] for r in g2] == [r["proof"] for r in g] and g2[-1]["window_state"] == g[-1]["window_state"]
    # matmul families spread over three more streams with SM budgets (bench --mm-streams): same bytes
    mm = [api.Context(0, torch.cuda.Stream()) for _ in range(3)]
    for c in [ctx] + mm:
        c.set_sm_budget(37)
    g3 = dfcn.prove_window(ctx, fs_seed("tiny"), fcn.fcn_header(shape), dfcn.upload_families(fams), relu_ctx=relu_ctx,
                           mm_ctxs=mm)
    ctx.set_sm_budget(0)
    assert [r["proof"] for r in g3] == [r["proof"] for r in g] and g3[-1]["window_state"] == g[-1]["window_state"]
    h3 = dfcn.prove_window_from_host(ctx, fs_seed("tiny"), fcn.fcn_header(shape), host, relu_ctx=relu_ctx, mm_ctxs=mm)
    assert [r["proof"] for r in h3] == [r["proof"] for r in g]


def test_fcn_tiny_merge_aux_vs_oracle(ctx, O):
    """The window with the aux-claim merge in every zkReLU family (D21): bit-exact against the oracle
    driver, and the synchronous zk_relu_merge gives the same bytes as the device-output one."""
    import torch
    from oracle import drivers
    from paper_2307_16273_b200 import api
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    shape = fcn.tiny_shape(steps=2, layers=3, width=16, batch=8, din=8, dout=4)
    trace = fcn.generate_trace(shape, x_bits=4, w_bits=4, y_bits=3)
    fams = fcn.assemble_families(shape, trace)
    o = drivers.fcn_prove(shape, fams, "tiny-merge", merge_aux=True)
    relu_ctx = api.Context(0, torch.cuda.Stream())
    g = dfcn.prove_window(ctx, fs_seed("tiny-merge"), fcn.fcn_header(shape), dfcn.upload_families(fams),
                          relu_ctx=relu_ctx, merge_aux=True)
    for gr, orr in zip(g, o):
        assert gr["msgs"] == orr["msgs"] and gr["finals"] == orr["finals"] and gr["state"] == orr["state"], gr["name"]
        if gr["kind"] == "relu":
            gm, om = gr["merge"], orr["merge"]
            assert gm["claim"] == om["claim"] and gm["msgs"] == om["msgs"] and gm["finals"] == om["finals"]
            assert gm["r"] == om["r"]
    assert g[-1]["window_state"] == o[-1]["window_state"]
    f = next(f for f in fams if not hasattr(f, "A"))
    t1 = api.Transcript(ctx, bytes(32))
    r1 = api.relu_prove(ctx, t1, dev(f.Z), dev(f.GA), f.Q, f.R)
    m1 = api.relu_merge(ctx, t1, dev(f.Z), dev(f.GA), f.Q, f.R, r1["point"], r1["finals"])
    t2 = api.Transcript(ctx, bytes(32))
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    ro = api.relu_prove_dev(ctx, t2, dev(f.Z), dev(f.GA), f.Q, f.R, flag)
    mo = api.relu_merge_dev(ctx, t2, dev(f.Z), dev(f.GA), f.Q, f.R, ro)
    pm = api.parse_relu_merge_out(mo.cpu().numpy().tobytes(), f.Q, f.R)
    assert pm["proof"] == m1["proof"] and pm["r"] == m1["r"] and t1.state() == t2.state()


def test_async_provers_match_sync(ctx):
    """zk_matmul_prove / zk_relu_prove_dev (device outputs, no host sync) give the bytes of the
    synchronous calls, back to back on one transcript; the range flag replaces ZK_ERR_RANGE."""
    import torch
    from paper_2307_16273_b200 import api
    A = uniform_range(21, 1, (4, 8, 32), -128, 128)
    B = uniform_range(21, 2, (4, 32, 16), -128, 128)
    Z = uniform_range(21, 3, (1 << 9,), -(1 << 15), 1 << 15)
    GA = uniform_range(21, 4, (1 << 9,), -(1 << 15), 1 << 15)
    seed = fs_seed("async")
    t1 = api.Transcript(ctx, seed)
    red = api.matmul_reduce(ctx, t1, dev(A), dev(B))
    sc = api.sumcheck_prove(ctx, t1, 2 + 5, 2, [red["At"], red["Bt"]], red["w"], red["claim"])
    rl = api.relu_prove(ctx, t1, dev(Z), dev(GA), 8, 8)
    t2 = api.Transcript(ctx, seed)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    mo = api.matmul_prove(ctx, t2, dev(A), dev(B))
    ro = api.relu_prove_dev(ctx, t2, dev(Z), dev(GA), 8, 8, flag)
    st = torch.empty(32, dtype=torch.uint8, device="cuda")
    t2.state_dev(st)
    pm = api.parse_matmul_out(mo.cpu().numpy().tobytes(), (2, 3, 5, 4))
    pr = api.parse_relu_out(ro.cpu().numpy().tobytes(), 9, 8, 8)
    assert pm["w"] == red["w"] and pm["u1"] == red["u1"] and pm["u3"] == red["u3"] and pm["claim"] == red["claim"]
    assert pm["proof"] == sc["proof"] and pm["r"] == sc["r"]
    assert pr["proof"] == rl["proof"] and pr["point"] == rl["point"]
    assert int(flag.item()) == 0
    assert st.cpu().numpy().tobytes() == t1.state()
    # out-of-range input: flag set, no exception
    Zb = Z.copy()
    Zb[5] = 1 << 20
    api.relu_prove_dev(ctx, api.Transcript(ctx, seed), dev(Zb), dev(GA), 8, 8, flag)
    assert int(flag.item()) & 1


# ---------------------------------------------------------------- §8(e) sharded sumcheck
SHARD_CASES = [(10, 10, 2), (12, 7, 2), (13, 13, 3), (9, 0, 1), (16, 16, 2)]


@pytest.mark.parametrize("m,n_eq,K", SHARD_CASES)
def test_shard_virtual_vs_oracle(ctx, O, m, n_eq, K):
    """G virtual shards on one device (same kernels as the multi-GPU path): transcript = single-device."""
    from paper_2307_16273_b200 import api, shard
    rng = random.Random(m + 100 * n_eq)
    tabs = [uniform_range(12, 31 * m + k, (1 << m,), -(1 << 15), 1 << 15) for k in range(K)]
    w = [rng.randrange(P) for _ in range(n_eq)]
    seed = fs_seed(f"shard-{m}-{n_eq}-{K}")
    o = O.sumcheck_prove(O.Transcript(seed), m, n_eq, [[int(v) % P for v in t] for t in tabs], w, None)
    for G in (1, 2, 4, 8):
        L = m - (G.bit_length() - 1)
        for switch in (0, 3, 40):
            trs = [api.Transcript(ctx, seed) for _ in range(G)]
            sess = [shard.ShardSession(ctx, trs[g], m, n_eq, [dev(t[g << L:(g + 1) << L]) for t in tabs], w, g, G)
                    for g in range(G)]
            res = shard.prove_virtual(sess, switch_log=switch)
            for g, r in enumerate(res):
                assert r["claim"] == o["claim"] and r["msgs"] == o["msgs"], (G, switch, g)
                assert r["finals"] == o["finals"] and r["r"] == o["r"], (G, switch, g)
            assert trs[0].state() == trs[-1].state()
            for s_ in sess:
                s_.close()


def test_shard_nccl_single_rank(ctx, O):
    """The torch.distributed/NCCL exchange path with one rank (the only GPU count gpurun grants)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2307_16273_b200 import api, shard
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m, n_eq = 14, 14
        A = uniform_range(13, 1, (1 << m,), -(1 << 15), 1 << 15)
        B = uniform_range(13, 2, (1 << m,), -(1 << 15), 1 << 15)
        rng = random.Random(3)
        w = [rng.randrange(P) for _ in range(n_eq)]
        seed = fs_seed("shard-nccl")
        o = O.sumcheck_prove(O.Transcript(seed), m, n_eq, [[int(v) % P for v in A], [int(v) % P for v in B]], w, None)
        tr = api.Transcript(ctx, seed)
        sess = shard.ShardSession(ctx, tr, m, n_eq, [dev(A), dev(B)], w, 0, 1)
        res = shard.prove(sess, shard.TorchComm(), switch_log=6)
        assert res["msgs"] == o["msgs"] and res["finals"] == o["finals"] and res["claim"] == o["claim"]
        # the exchange owned by the library (zk_ctx_attach_nccl + zk_sc_shard_prove_nccl), two switch points
        c2 = api.Context(0)
        assert shard.attach_nccl(c2) == (0, 1)
        for sw in (6, 20):
            tr2 = api.Transcript(c2, seed)
            s2 = shard.ShardSession(c2, tr2, m, n_eq, [dev(A), dev(B)], w, 0, 1)
            r2 = shard.prove_nccl(s2, switch_log=sw)
            assert r2["msgs"] == o["msgs"] and r2["finals"] == o["finals"] and r2["claim"] == o["claim"]
            s2.close()
            tr2.close()
    finally:
        dist.destroy_process_group()


# ---------------------------------------------------------------- BASELINE workloads at full size
@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_fcn_window_full_size_vs_oracle(ctx, O, cfg):
    """C3 (one training step of the uniform 8 x 1024^2 FCN) and C4 (the bench.py workload: a T' = 16
    window of the paper's 10M FCN) at full size in the bench's launch configuration (zkReLU on a second
    stream, matmul families over four budgeted streams): every matmul family is bit-exact against the
    oracle's own proof (brute-force restriction, claim = brute-force MLE of the exact integer product),
    the 2^23-entry zkReLU family is accepted by the oracle verifier (claims = brute-force MLEs of Z, A,
    G_A, G_Z; finals = brute-force aux MLEs of the bits), and every family's and the window's
    transcript state equal the oracle's (D3d)."""
    import os
    import torch
    from paper_2307_16273_b200 import api
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    from synth.prng import DATA_SEED
    O.set_threads(len(os.sched_getaffinity(0)))
    shape = fcn.C4_SHAPE if cfg == "C4" else fcn.C3_SHAPE
    seed_name = "C4-rank0" if cfg == "C4" else "C3"
    fams = fcn.assemble_families(shape, fcn.generate_trace(shape, seed=DATA_SEED))
    relu_ctx = api.Context(0, torch.cuda.Stream())
    mm = [api.Context(0, torch.cuda.Stream()) for _ in range(3)]
    for c in [ctx] + mm:
        c.set_sm_budget(37)
    merge = cfg == "C4"   # C4 also with the aux-claim merge of N1 (D21) in the zkReLU family
    g = dfcn.prove_window(ctx, fs_seed(seed_name), fcn.fcn_header(shape), dfcn.upload_families(fams),
                          relu_ctx=relu_ctx, mm_ctxs=mm, merge_aux=merge)
    ctx.set_sm_budget(0)
    W = O.Transcript(fs_seed(seed_name))
    W.absorb("fcn/hdr", fcn.fcn_header(shape))
    forks = []
    for f in fams:
        W.absorb("fcn/fam", f.name.encode())
        forks.append(O.Transcript(W.challenges("fcn/fork", 1)[0].to_bytes(32, "little")))
    for f, T, gr in zip(fams, forks, g):
        if hasattr(f, "A"):
            o = O.matmul_prove(T, f.A, f.B, f.transA, f.transB)
            assert (gr["w"], gr["u1"], gr["u3"], gr["claim"]) == (o["w"], o["u1"], o["u3"], o["claim"]), f.name
            assert gr["msgs"] == o["msgs"] and gr["finals"] == o["finals"], f.name
        else:
            assert O.relu_verify(T, f.Z, f.GA, f.Q, f.R, gr["claims"], gr["msgs"], gr["finals"]) == 0, f.name
            if merge:   # the merge's claim from the verified finals, then its round identities
                gm = gr["merge"]
                rho = T.challenges("relu/merge", 1)[0]
                f0, f1, f2 = gr["finals"]
                assert gm["claim"] == (f0 + rho * f1 + rho * rho * f2) % P
                assert O.sumcheck_verify(T, 6, 0, 2, [], gm["claim"], gm["msgs"], gm["finals"]) == 0
        assert gr["state"] == T.state(), f.name
    for T in forks:
        W.absorb("fcn/join", T.state())
    assert g[-1]["window_state"] == W.state()
    # the library's own host verifier (N3, D23) accepts the GPU window: every family, the joins
    from paper_2307_16273_b200 import verify
    vo = verify.verify_window(fs_seed(seed_name), fcn.fcn_header(shape), fams, g)
    assert [v["point"] for v in vo] == [gr["r"] if hasattr(f, "A") else gr["point"] for f, gr in zip(fams, g)]


@pytest.mark.slow
@pytest.mark.parametrize("m", [24, 26, 28, 30])
def test_c5_large_properties(ctx, O, m):
    """C5 (BASELINE configs[4]: the aggregated Hadamard statement sum_x eq(w,x) A(x) B(x)) at
    the sweep sizes 2^24 ... 2^30, too large for a full oracle prover run: inputs generated on the device
    by the counter PRNG (checked against the numpy generator at both ends), the oracle verifier replays
    the transcript and checks every round identity, the finals are checked against
    brute-force MLEs of A and B at r, and the claim against the brute-force MLE of the integer
    product table at w (|A B| < 2^30); the library's host verifier ends in the prover's state."""
    import os
    from paper_2307_16273_b200 import api, verify
    from synth.prng import DATA_SEED, uniform_bits, uniform_range_torch
    O.set_threads(len(os.sched_getaffinity(0)))
    n = 1 << m
    dA = uniform_range_torch(DATA_SEED, 21, n, -(1 << 15), 1 << 15, "cuda")
    dB = uniform_range_torch(DATA_SEED, 22, n, -(1 << 15), 1 << 15, "cuda")
    for tid, d in ((21, dA), (22, dB)):
        ref = uniform_range(DATA_SEED, tid, (1 << 12,), -(1 << 15), 1 << 15)
        assert np.array_equal(d[:1 << 12].cpu().numpy(), ref)
        end = uniform_bits(DATA_SEED, tid, 1 << 12, -(1 << 15), 16, offset=n - (1 << 12)).astype(np.int32)
        assert np.array_equal(d[n - (1 << 12):].cpu().numpy(), end)
    tr = api.Transcript(ctx, fs_seed(f"C5-m{m}"))
    tr.absorb("c5/hdr", m.to_bytes(4, "little"))
    w = tr.challenges("c5/w", m)
    g = api.sumcheck_prove(ctx, tr, m, m, [dA, dB], w)
    A, B = dA.cpu().numpy(), dB.cpu().numpy()
    del dA, dB
    torch.cuda.empty_cache()
    ot = O.Transcript(fs_seed(f"C5-m{m}"))
    ot.absorb("c5/hdr", m.to_bytes(4, "little"))
    assert ot.challenges("c5/w", m) == w
    assert g["finals"] == [O.mle_i32(A, g["r"]), O.mle_i32(B, g["r"])]
    assert O.sumcheck_verify(ot, m, m, 2, w, g["claim"], g["msgs"], g["finals"]) == 0
    assert ot.state() == tr.state()
    np.multiply(A, B, out=A)                     # |A B| <= 2^30: exact in int32
    assert g["claim"] == O.mle_i32(A, w)
    H = verify.HostTranscript(seed=fs_seed(f"C5-m{m}"))
    H.absorb("c5/hdr", m.to_bytes(4, "little"))
    assert H.challenges("c5/w", m) == w
    assert verify.verify_sumcheck(H, g["proof"], w, shape=(m, m, 2)) == g["r"] and H.state() == tr.state()


@pytest.mark.parametrize("m", [22])
def test_c5_bench_size_vs_oracle(ctx, O, m):
    """C5 at the smallest BASELINE sweep size through the path bench.py --config C5 times (int32 tables
    embedded in round 0, grouped and flat factored rounds, persistent tail): bit-exact."""
    from oracle import drivers
    from paper_2307_16273_b200 import api
    A, B = drivers.c5_inputs(m)
    o = drivers.c5_prove(m)
    tr = api.Transcript(ctx, fs_seed(f"C5-m{m}"))
    tr.absorb("c5/hdr", m.to_bytes(4, "little"))
    w = tr.challenges("c5/w", m)
    g = api.sumcheck_prove(ctx, tr, m, m, [dev(A), dev(B)], w)
    assert g["claim"] == o["claim"] and g["msgs"] == o["msgs"] and g["finals"] == o["finals"]


# ---------------------------------------------------------------- SURVEY §8(f) N1
@pytest.mark.parametrize("n,d,nks", [(3, 2, [3, 2, 1]), (6, 5, [6, 5]), (10, 8, [10, 9, 0]), (14, 4, [13, 14])])
def test_reindex_vs_oracle(ctx, O, n, d, nks):
    """Re-indexing sumcheck (Eq. sc-reindex): transcript bit-exact against the oracle, views with empty
    slots and several sizes (the larger ones through the factored round kernel)."""
    from paper_2307_16273_b200 import api
    rng = random.Random(1000 + n)
    X = uniform_range(13, n + d, (1 << n, 1 << d), -(1 << 15), 1 << 15)
    u = [rng.randrange(P) for _ in range(d)]
    views = []
    for nk in nks:
        pick = rng.sample(range(1 << n), min(1 << nk, 1 << n))
        mp = pick + [-1] * ((1 << nk) - len(pick))
        rng.shuffle(mp)
        views.append((mp, [rng.randrange(P) for _ in range(nk)]))
    claims = [rng.randrange(P) for _ in views]      # any claims: the transcript is still determined
    seed = fs_seed(f"rx-gpu-{n}-{d}")
    o = O.reindex_prove(O.Transcript(seed), X, views, u, claims)
    g = api.reindex_prove(ctx, api.Transcript(ctx, seed), dev(X), views, u, claims)
    assert g["claim"] == o["claim"] and g["msgs"] == o["msgs"] and g["finals"] == o["finals"] and g["r"] == o["r"]


def test_reindex_rejects_bad_maps(ctx):
    from paper_2307_16273_b200 import api
    X = dev(uniform_range(13, 1, (8, 4), -8, 8))
    for mp in ([0, 0], [0, 9]):
        with pytest.raises(api.ZkError):
            api.reindex_prove(ctx, api.Transcript(ctx, bytes(32)), X, [(mp, [5])], [1, 2], [3])


@pytest.mark.parametrize("Q,R,logD", [(4, 2, 3), (16, 16, 8), (8, 8, 12), (16, 16, 16)])
def test_relu_merge_vs_oracle(ctx, O, Q, R, logD):
    """zkReLU prove then the aux-claim merge on the same transcript: bit-exact against the oracle."""
    from paper_2307_16273_b200 import api
    half = 1 << (Q + R - 1)
    Z = uniform_range(14, logD + Q, (1 << logD,), -half, half)
    GA = uniform_range(14, logD + R + 1, (1 << logD,), -half, half)
    seed = fs_seed(f"merge-gpu-{Q}-{R}-{logD}")
    ot = O.Transcript(seed)
    orr = O.relu_prove(ot, Z, GA, Q, R)
    om = O.relu_merge(ot, Z, GA, Q, R, orr["point"], orr["finals"])
    gt = api.Transcript(ctx, seed)
    gr = api.relu_prove(ctx, gt, dev(Z), dev(GA), Q, R)
    assert gr["finals"] == orr["finals"]
    gm = api.relu_merge(ctx, gt, dev(Z), dev(GA), Q, R, gr["point"], gr["finals"])
    assert gm["claim"] == om["claim"] and gm["msgs"] == om["msgs"] and gm["finals"] == om["finals"]
    assert gt.state() == ot.state()


def test_relu_merge_c4_size(ctx, O):
    """The merge at the C4 zkReLU size (2^23 entries): the merged claim equals aux~(r_s, v, r_j) built
    from the oracle's brute-force MLEs of the 64 bit planes, and the oracle verifier accepts the merge
    sumcheck's round identities."""
    import os
    from paper_2307_16273_b200 import api
    O.set_threads(len(os.sched_getaffinity(0)))
    logD = 23
    Z = uniform_range(15, 1, (1 << logD,), -(1 << 31), 1 << 31)
    GA = uniform_range(15, 2, (1 << logD,), -(1 << 31), 1 << 31)
    rng = random.Random(9)
    point = [rng.randrange(P) for _ in range(5 + logD)]
    w, v = point[:5], point[5:]
    planes = [[O.mle_i32((((word.astype(np.int64) & 0xFFFFFFFF) >> j) & 1).astype(np.int32), v) for j in range(32)]
              for word in (Z, GA)]                    # aux~(s, v, j) at Boolean j
    beta5 = lambda x, j: O.beta(x, [(j >> t) & 1 for t in range(5)])
    ew = [beta5(w, j) for j in range(32)]
    f0 = sum(e * p for e, p in zip(ew, planes[0])) % P
    f1 = sum(e * p for e, p in zip(ew, planes[1])) % P
    f2 = planes[0][31]
    seed = fs_seed("merge-c4")
    gm = api.relu_merge(ctx, api.Transcript(ctx, seed), dev(Z), dev(GA), 16, 16, point, [f0, f1, f2])
    rj, rs = gm["r"][:5], gm["r"][5]
    ej = [beta5(rj, j) for j in range(32)]
    t0 = sum(e * p for e, p in zip(ej, planes[0])) % P
    t1 = sum(e * p for e, p in zip(ej, planes[1])) % P
    assert gm["finals"][0] == ((1 - rs) * t0 + rs * t1) % P
    tr = O.Transcript(seed)
    rho = tr.challenges("relu/merge", 1)[0]
    claim = (f0 + rho * f1 + rho * rho * f2) % P
    assert gm["claim"] == claim
    assert O.sumcheck_verify(tr, 6, 0, 2, [], claim, gm["msgs"], gm["finals"]) == 0


# ---------------------------------------------------------------- SURVEY §8(f) N2
@pytest.mark.parametrize("m", [1, 5, 12, 17, 20])
def test_hadamard_zero_vs_oracle(ctx, O, m):
    """Protocol 2's zero form (D22): bit-exact against the oracle, for a true statement Y = A (.) B and for a
    false one (one entry of Y off by one: the proof is still determined and must match)."""
    from paper_2307_16273_b200 import api
    A = uniform_range(33, m, (1 << m,), -(1 << 15), 1 << 15)
    B = uniform_range(33, m + 50, (1 << m,), -(1 << 15), 1 << 15)
    for bad in (False, True):
        Y = (A.astype(np.int64) * B).astype(np.int32)
        if bad:
            Y[(1 << m) // 3] += 1
        seed = fs_seed(f"hd-gpu-{m}-{bad}")
        o = O.zero_sumcheck_prove(O.Transcript(seed), Y, A, B)
        g = api.hadamard_zero_prove(ctx, api.Transcript(ctx, seed), dev(Y), dev(A), dev(B))
        assert g["w"] == o["w"] and g["msgs"] == o["msgs"] and g["r"] == o["r"] and g["finals"] == o["finals"]
        first = ((1 - g["w"][0]) * g["msgs"][0][0] + g["w"][0] * g["msgs"][0][1]) % P
        assert (first == 0) == (not bad)


@pytest.mark.parametrize("nrows,cols", [(1024, 8), (1024 + 24, 16), (18944, 64), (4096, 1024), (131072, 1024), (3000, 4096)])
def test_rowdot_tensor_cores_vs_oracle(ctx, O, nrows, cols):
    """The matmul restriction's row dots (row r of M against eq(u, .)) on the tensor cores
    (int8 GEMM over the bytes of the int32 matrix, restrict_tc.cu) and on the CUDA cores, each against
    the oracle's brute-force MLE of the row: the full int32 range (rows 0/1 at -2^31 and 2^31-1), ragged
    row counts, several tiles per CTA; every row up to 4096 rows, else the first/last 512 and 512 random."""
    from paper_2307_16273_b200._lib import lib
    from paper_2307_16273_b200 import api
    rng = random.Random(nrows + cols)
    M = torch.randint(-2 ** 31, 2 ** 31, (nrows, cols), dtype=torch.int64, generator=torch.Generator().manual_seed(nrows)).to(torch.int32)
    M[0, :] = -2 ** 31
    M[1, :] = 2 ** 31 - 1
    Mh = M.numpy()
    pt = [rng.randrange(P) for _ in range(cols.bit_length() - 1)]
    rows = list(range(nrows)) if nrows <= 4096 else sorted(set(range(512)) | set(range(nrows - 512, nrows))
                                                           | set(rng.sample(range(nrows), 512)))
    O.set_threads(1)
    want = [O.mle_i32(Mh[r], pt) for r in rows]
    for tc in (0, 1, 2):   # CUDA cores; tensor cores with the cp.async producer; with the TMA producer
        o = torch.zeros((nrows, 32), dtype=torch.uint8, device="cuda")
        ctx.check(lib().zk_diag_rowdot(ctx.h, M.cuda().data_ptr(), nrows, cols, api._fr_buf(pt), o.data_ptr(), tc))
        got = api.fr_table_to_ints(ctx, o)
        assert [got[r] for r in rows] == want, f"use_tc={tc}"


# ---------------------------------------------------------------- N2: the loss-gradient family (D24)
@pytest.mark.parametrize("m", [1, 10, 16])
def test_loss_grad_vs_oracle(ctx, O, m):
    """zk_loss_grad_prove against the oracle: the point, the three claims and the transcript state
    bit-exact; the library's host verifier accepts; the identity fails for a false G_Z."""
    from paper_2307_16273_b200 import api, verify
    Z = uniform_range(44, m, (1 << m,), -(1 << 30), 1 << 30)
    Y = uniform_range(44, m + 30, (1 << m,), -(1 << 30), 1 << 30)
    G = (Z.astype(np.int64) - Y).astype(np.int32)
    seed = fs_seed(f"lg-gpu-{m}")
    T = O.Transcript(seed)
    o = O.loss_grad_prove(T, G, Z, Y)
    tr = api.Transcript(ctx, seed)
    g = api.loss_grad_prove(ctx, tr, dev(G), dev(Z), dev(Y))
    assert g == o and tr.state() == T.state()
    assert verify.verify_loss_grad(verify.HostTranscript(seed=seed), m, g["claims"]) == g["u"]
    G[0] += 1
    gb = api.loss_grad_prove(ctx, api.Transcript(ctx, seed), dev(G), dev(Z), dev(Y))
    assert gb["claims"][0] != (gb["claims"][1] - gb["claims"][2]) % P


def test_readme_flow_host_verified(ctx, O):
    """The README's usage: a matmul reduction + product sumcheck and a zkReLU proof on one transcript,
    then the host verifiers replaying the same transcript accept both and end in the prover's state."""
    from paper_2307_16273_b200 import api, verify
    A = uniform_range(9, 1, (4, 8, 16), -(1 << 15), 1 << 15)
    B = uniform_range(9, 2, (4, 16, 32), -(1 << 15), 1 << 15)
    Z = uniform_range(9, 3, (1 << 12,), -(1 << 31), 1 << 31)
    GA = uniform_range(9, 4, (1 << 12,), -(1 << 31), 1 << 31)
    tr = api.Transcript(ctx, b"\0" * 32)
    red = api.matmul_reduce(ctx, tr, dev(A), dev(B))
    logN, logD2 = len(red["w"]), 4
    proof = api.sumcheck_prove(ctx, tr, logN + logD2, logN, [red["At"], red["Bt"]], red["w"], red["claim"])
    relu = api.relu_prove(ctx, tr, dev(Z), dev(GA), 16, 16)
    H = verify.HostTranscript(seed=b"\0" * 32)
    logs = (logN, len(red["u1"]), logD2, len(red["u3"]))
    assert verify.verify_matmul(H, logs, dict(red, proof=proof["proof"]))["r"] == proof["r"]
    assert verify.verify_relu(H, relu["proof"], (12, 16, 16))["point"] == relu["point"]
    assert H.state() == tr.state()


def test_e2e_int16_transport_same_proofs(ctx):
    """prove_windows_from_host with the stacks whose entries fit 16 bits shipped as int16 (zk_widen_i16 on
    the device) gives the bytes of the device-resident window (the same int32 tensors are proved)."""
    import numpy as np
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    shape = fcn.tiny_shape(steps=2, layers=5, width=64, batch=16, din=128, dout=16)
    fams = fcn.assemble_families(shape, fcn.generate_trace(shape))
    seed, hdr = fs_seed("e2e-i16"), fcn.fcn_header(shape)
    g = dfcn.prove_window(ctx, seed, hdr, dfcn.upload_families(fams))
    padded = []

    def host(a):   # as bench.py: int16 where the entries fit, trailing zero slots not shipped (HostStack)
        small = int(a.max()) < (1 << 15) and int(a.min()) >= -(1 << 15)
        nz = np.flatnonzero(a.reshape(a.shape[0], -1).any(axis=1)) if a.ndim > 1 else np.array([0])
        n = int(nz[-1]) + 1 if nz.size else 1
        body = a[:n] if a.ndim > 1 else a
        t = torch.from_numpy(np.ascontiguousarray(body.astype(np.int16) if small else body)).pin_memory()
        if a.ndim > 1 and n < a.shape[0]:
            padded.append(a.shape)
            return dfcn.HostStack(t, a.shape)
        return t
    hf = [dfcn.DeviceFamily(f.name, "matmul", A=host(f.A), B=host(f.B), trans_a=f.transA, trans_b=f.transB)
          if hasattr(f, "A") else dfcn.DeviceFamily(f.name, "relu", Z=host(f.Z), GA=host(f.GA), Q=f.Q, R=f.R) for f in fams]
    assert any(t.dtype == torch.int16 for f in hf for t in (f.A, f.B, f.Z, f.GA) if t is not None)
    assert padded   # some stacks travel without their zero padding slots
    h = dfcn.prove_windows_from_host(ctx, [(seed, hdr, hf)])[0]
    assert [r["proof"] for r in h] == [r["proof"] for r in g]
    assert h[-1]["window_state"] == g[-1]["window_state"]
    x = torch.arange(-(1 << 15), (1 << 15), 37, dtype=torch.int16)
    from paper_2307_16273_b200 import api
    y = api.widen_i16(ctx, x.cuda())
    assert torch.equal(y.cpu(), x.to(torch.int32))


def test_e2e_delta_transport_same_proofs(ctx):
    """Weight stacks shipped as their first slots (int16) + int8 slot differences (fcn.delta_stack, rebuilt by
    zk_undelta_i8 on the device) give the bytes of the device-resident window; zk_undelta_i8 rebuilds a random
    stack exactly (padding slots stay zero)."""
    import numpy as np
    from paper_2307_16273_b200 import api
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    shape = fcn.tiny_shape(steps=2, layers=5, width=64, batch=16, din=128, dout=16)
    fams = fcn.assemble_families(shape, fcn.generate_trace(shape))
    seed, hdr = fs_seed("e2e-delta"), fcn.fcn_header(shape)
    g = dfcn.prove_window(ctx, seed, hdr, dfcn.upload_families(fams))
    deltas = []

    def host(a):
        if a.ndim > 1:
            nz = np.flatnonzero(a.reshape(a.shape[0], -1).any(axis=1))
            ds = dfcn.delta_stack(a, int(nz[-1]) + 1 if nz.size else 1)
            if ds is not None:
                deltas.append(ds)
                return ds
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hf = [dfcn.DeviceFamily(f.name, "matmul", A=host(f.A), B=host(f.B), trans_a=f.transA, trans_b=f.transB)
          if hasattr(f, "A") else dfcn.DeviceFamily(f.name, "relu", Z=host(f.Z), GA=host(f.GA), Q=f.Q, R=f.R) for f in fams]
    assert any(d.L > 1 for d in deltas)   # the hidden-layer weight stack: stride = layers per step
    h = dfcn.prove_windows_from_host(ctx, [(seed, hdr, hf)] * 2)
    for w in h:
        assert [r["proof"] for r in w] == [r["proof"] for r in g]
    rng = np.random.default_rng(5)
    a = np.zeros((16, 6, 8), np.int32)
    a[:3] = rng.integers(-30000, 30000, (3, 6, 8))
    for s in range(3, 13):
        a[s] = a[s - 3] + rng.integers(-128, 128, (6, 8))
    ds = dfcn.delta_stack(a, 13)
    assert ds is not None and ds.L == 3
    out = torch.full((16, 6, 8), -1, dtype=torch.int32, device="cuda")
    out[13:].zero_()
    api.undelta_i8(ctx, ds.base.cuda(), ds.delta.cuda(), 3, 13, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), a)
