"""Pins for the oracle's eq/MLE, product sumcheck and matmul reduction (-m "not gpu").

Pinned against: SPEC worked examples,
closed forms (one-variable MLE is the line through two points; beta is the
indicator on Boolean points and sums to 1), the round identities of
Protocols 2-3, the final check against brute-force
MLE, Eq. (5)'s single-instance compression, the stacking identity
(S:L151), integer matrix products, exhaustive tiny inputs, and tampering.
"""
import itertools
import random

import numpy as np
import pytest

from synth.prng import uniform_range

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def rnd(rng, n):
    return [rng.randrange(P) for _ in range(n)]


def test_beta_spec_and_indicator(oracle_lib):
    O = oracle_lib
    assert O.beta([2, 3], [1, 0]) == (-4) % P
    assert O.beta([0, 1], [0, 1]) == 1 and O.beta([0, 1], [1, 1]) == 0
    for k in range(0, 5):                                              # Boolean points: indicator
        for b in range(1 << k):
            bits = [(b >> t) & 1 for t in range(k)]
            tab = O.eq_table(bits)
            assert tab == [1 if x == b else 0 for x in range(1 << k)]


def test_eq_table_sums_to_one_and_multiplicative(oracle_lib):
    O = oracle_lib
    rng = random.Random(1)
    u, v = rnd(rng, 3), rnd(rng, 2)
    t = O.eq_table(u)
    assert sum(t) % P == 1
    # beta(u||v, b||c) = beta(u,b) beta(v,c): the table over u||v is the outer product, LSB first (D2)
    tuv, tv = O.eq_table(u + v), O.eq_table(v)
    for x in range(32):
        assert tuv[x] == t[x & 7] * tv[x >> 3] % P


def test_mle_spec_and_line(oracle_lib):
    O = oracle_lib
    assert O.mle_fr([5, 7], [0]) == 5 and O.mle_fr([5, 7], [1]) == 7 and O.mle_fr([5, 7], [2]) == 9
    rng = random.Random(2)
    for _ in range(20):
        a, b, u = rnd(rng, 3)
        assert O.mle_fr([a, b], [u]) == (a + u * (b - a)) % P


def test_mle_boolean_points_exhaustive_256(oracle_lib):
    O = oracle_lib
    rng = random.Random(3)
    tab = rnd(rng, 256)
    for b in range(256):
        assert O.mle_fr(tab, [(b >> t) & 1 for t in range(8)]) == tab[b]


def test_mle_multilinear_in_each_coordinate(oracle_lib):
    O = oracle_lib
    rng = random.Random(4)
    tab = rnd(rng, 32)
    u = rnd(rng, 5)
    for t in range(5):
        x = u[t]
        f0 = O.mle_fr(tab, u[:t] + [0] + u[t + 1:])
        f1 = O.mle_fr(tab, u[:t] + [1] + u[t + 1:])
        assert O.mle_fr(tab, u) == ((1 - x) * f0 + x * f1) % P


def test_mle_i32_matches_embedding(oracle_lib):
    O = oracle_lib
    rng = random.Random(5)
    t = uniform_range(5, 5, (64,), -(1 << 31), 1 << 31)
    u = rnd(rng, 6)
    assert O.mle_i32(t, u) == O.mle_fr([int(v) % P for v in t], u)


def test_stacking_identity(oracle_lib):
    # Z~(w, u) = sum_i beta(w, i) Z^(i)~(u); stack axis = high bits of the flat index
    O = oracle_lib
    rng = random.Random(6)
    inst = [rnd(rng, 8) for _ in range(4)]
    w, u = rnd(rng, 2), rnd(rng, 3)
    stacked = [v for t in inst for v in t]
    lhs = O.mle_fr(stacked, u + w)
    ew = O.eq_table(w)
    assert lhs == sum(ew[i] * O.mle_fr(inst[i], u) for i in range(4)) % P


def test_sumcheck_spec_sum(oracle_lib):
    O = oracle_lib
    res = O.sumcheck_prove(O.Transcript(bytes(32)), 2, 0, [[1, 2, 3, 4]], [])
    assert res["claim"] == 10
    assert res["msgs"][0][0] + res["msgs"][0][1] == 10


def _brute_claim(tables, w, n_eq):
    m = len(tables[0]).bit_length() - 1
    tot = 0
    for x in range(1 << m):
        e = 1
        for t in range(n_eq):
            e = e * (w[t] if (x >> t) & 1 else 1 - w[t]) % P
        p = e
        for tb in tables:
            p = p * tb[x] % P
        tot += p
    return tot % P


def test_sumcheck_one_round_closed_form(oracle_lib):
    # m = 1: the only message is prod_k (T_k[0] + X (T_k[1] - T_k[0])) at X = 0..K, in both forms
    O = oracle_lib
    rng = random.Random(8)
    for K in (1, 2, 3):
        for n_eq in (0, 1):
            T = [rnd(rng, 2) for _ in range(K)]
            w = rnd(rng, n_eq)
            res = O.sumcheck_prove(O.Transcript(bytes(32)), 1, n_eq, T, w)
            for X in range(K + 1):
                want = 1
                for t in T:
                    want = want * (t[0] + X * (t[1] - t[0])) % P
                assert res["msgs"][0][X] == want
            assert res["finals"] == [(t[0] + res["r"][0] * (t[1] - t[0])) % P for t in T]


def test_sumcheck_exhaustive_m2(oracle_lib):
    """m = 2, K = 2, entries in {0, 1, 2, p-1}: every A against 16 B patterns, n_eq in {0, 1, 2}."""
    O = oracle_lib
    vals = [0, 1, 2, P - 1]
    rng = random.Random(9)
    Bs = [list(b) for b in rng.sample(list(itertools.product(vals, repeat=4)), 16)]
    w = rnd(rng, 2)
    cnt = 0
    for A in itertools.product(vals, repeat=4):
        A = list(A)
        for bi, Bt in enumerate(Bs):
            n_eq = (cnt % 3)
            cnt += 1
            res = O.sumcheck_prove(O.Transcript(bytes(32)), 2, n_eq, [A, Bt], w[:n_eq])
            assert res["claim"] == _brute_claim([A, Bt], w, n_eq)
            st = O.sumcheck_verify(O.Transcript(bytes(32)), 2, n_eq, 2, w[:n_eq], res["claim"], res["msgs"],
                                   res["finals"], [A, Bt])
            assert st == 0


@pytest.mark.parametrize("m,n_eq,K", [(6, 6, 2), (7, 3, 2), (8, 0, 3), (5, 5, 1), (9, 4, 3), (10, 10, 2)])
def test_sumcheck_random_accepts(oracle_lib, m, n_eq, K):
    O = oracle_lib
    rng = random.Random(m * 100 + n_eq * 10 + K)
    T = [rnd(rng, 1 << m) for _ in range(K)]
    w = rnd(rng, n_eq)
    res = O.sumcheck_prove(O.Transcript(b"\x01" * 32), m, n_eq, T, w)
    assert res["claim"] == _brute_claim(T, w, n_eq)
    assert O.sumcheck_verify(O.Transcript(b"\x01" * 32), m, n_eq, K, w, res["claim"], res["msgs"], res["finals"], T) == 0


def test_sumcheck_tamper_rejected(oracle_lib):
    O = oracle_lib
    rng = random.Random(11)
    m, n_eq, K = 6, 3, 2
    rejected = 0
    for trial in range(200):
        T = [rnd(rng, 1 << m) for _ in range(K)]
        w = rnd(rng, n_eq)
        res = O.sumcheck_prove(O.Transcript(bytes(32)), m, n_eq, T, w)
        kind = trial % 3
        msgs = [list(r) for r in res["msgs"]]
        fin = list(res["finals"])
        T2 = [list(t) for t in T]
        if kind == 0:
            t, x = rng.randrange(m), rng.randrange(K + 1)
            msgs[t][x] = (msgs[t][x] + 1) % P
        elif kind == 1:
            fin[0] = (fin[0] + 1) % P
        else:     # a corrupted input entry: the honest transcript no longer matches the table's MLE
            T2[0][rng.randrange(1 << m)] ^= 1
        st = O.sumcheck_verify(O.Transcript(bytes(32)), m, n_eq, K, w, res["claim"], msgs, fin, T2)
        rejected += st != 0
    assert rejected == 200


def test_aggregation_compresses_to_single_instance(oracle_lib):
    """Eq. (5): after the log N stack rounds, the running claim equals
    sum_k At~(v, k) Bt~(v, k) with v the stack challenges — the single-instance sumcheck."""
    O = oracle_lib
    logN, logD2 = 2, 3
    A = uniform_range(1, 31, (4, 2, 8), -(1 << 15), 1 << 15)
    B = uniform_range(1, 32, (4, 8, 2), -(1 << 15), 1 << 15)
    res = O.matmul_prove(O.Transcript(bytes(32)), A, B)
    N, D2 = 1 << logN, 1 << logD2
    c = res["claim"]
    for t in range(logN):
        ev = res["msgs"][t]
        r = res["r"][t]
        # Lagrange through 0,1,2
        c = (ev[0] * (r - 1) * (r - 2) * pow(2, -1, P) - ev[1] * r * (r - 2) + ev[2] * r * (r - 1) * pow(2, -1, P)) % P
    v = res["r"][:logN]
    s = 0
    for k in range(D2):
        s += O.mle_fr(res["At"][k * N:(k + 1) * N], v) * O.mle_fr(res["Bt"][k * N:(k + 1) * N], v)
    assert c == s % P


def _int_claim(Y, w, u1, u3):
    O_ = None
    N, D1, D3 = Y.shape
    tot = 0
    for n in range(N):
        for a in range(D1):
            for c_ in range(D3):
                e = 1
                for t, x in enumerate(w):
                    e = e * (x if (n >> t) & 1 else 1 - x) % P
                for t, x in enumerate(u1):
                    e = e * (x if (a >> t) & 1 else 1 - x) % P
                for t, x in enumerate(u3):
                    e = e * (x if (c_ >> t) & 1 else 1 - x) % P
                tot += e * int(Y[n, a, c_])
    return tot % P


def test_matmul_spec_example(oracle_lib):
    O = oracle_lib
    A = np.array([[[1, 2], [3, 4]]], dtype=np.int32)
    B = np.array([[[5, 6], [7, 8]]], dtype=np.int32)
    res = O.matmul_prove(O.Transcript(bytes(32)), A, B)
    Y = np.array([[19, 22], [43, 50]], dtype=np.int32)
    # claim = Y~(u1, u3): point order for a row-major matrix is (col bits, row bits) (D2)
    assert res["claim"] == O.mle_i32(Y.reshape(-1), res["u3"] + res["u1"])


@pytest.mark.parametrize("transA,transB", [(False, False), (True, False), (False, True), (True, True)])
def test_matmul_identity_and_verify(oracle_lib, transA, transB):
    O = oracle_lib
    N, D1, D2, D3 = 4, 8, 16, 4
    A = uniform_range(2, 41, (N, D1, D2), -(1 << 15), 1 << 15)
    B = uniform_range(2, 42, (N, D2, D3), -(1 << 15), 1 << 15)
    Y = np.einsum("nak,nkc->nac", A.astype(np.int64), B.astype(np.int64))
    As = np.ascontiguousarray(A.transpose(0, 2, 1)) if transA else A
    Bs = np.ascontiguousarray(B.transpose(0, 2, 1)) if transB else B
    seed = bytes(range(32))
    res = O.matmul_prove(O.Transcript(seed), As, Bs, transA, transB)
    assert res["claim"] == _int_claim(Y, res["w"], res["u1"], res["u3"])   # C(r1,r2) from integers
    # matmul identity through the restriction route: claim = sum_{k,n} beta(w,n) At[k][n] Bt[k][n]
    ew = O.eq_table(res["w"])
    s = sum(ew[i % N] * res["At"][i] * res["Bt"][i] for i in range(N * D2)) % P
    assert s == res["claim"]
    # replay + verify, finals against brute-force MLE of the restricted tables
    tr = O.Transcript(seed)
    tr.absorb("mm/hdr", b"".join(int(x).to_bytes(4, "little") for x in res["logs"]))
    tr.challenges("mm/w", 2), tr.challenges("mm/u1", 3), tr.challenges("mm/u3", 2)
    st = O.sumcheck_verify(tr, 2 + 4, 2, 2, res["w"], res["claim"], res["msgs"], res["finals"], [res["At"], res["Bt"]])
    assert st == 0
    # the final on At equals the MLE of A at (r_k, u1, r_n) — the claim handed to A's commitment
    r_n, r_k = res["r"][:2], res["r"][2:]
    assert res["finals"][0] == O.mle_i32(A.reshape(-1), r_k + res["u1"] + r_n)
    assert res["finals"][1] == O.mle_i32(B.reshape(-1), res["u3"] + r_k + r_n)


def test_aggregated_equals_individual(oracle_lib):
    # aggregated claim = sum_n beta(w, n) * claim of instance n at the same (u1, u3)
    O = oracle_lib
    A = uniform_range(3, 51, (4, 4, 4), -(1 << 15), 1 << 15)
    B = uniform_range(3, 52, (4, 4, 4), -(1 << 15), 1 << 15)
    res = O.matmul_prove(O.Transcript(bytes(32)), A, B)
    ew = O.eq_table(res["w"])
    tot = 0
    for n in range(4):
        Yn = (A[n].astype(np.int64) @ B[n].astype(np.int64)).reshape(-1)
        tot += ew[n] * O.mle_fr([int(v) % P for v in Yn], res["u3"] + res["u1"])
    assert tot % P == res["claim"]
