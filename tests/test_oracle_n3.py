"""Pins for the oracle's N3 pieces (-m "not gpu"): the claim merge of DESIGN.md D25 (Eq. sc-reindex,
P:L262-270, in its general form) and the chained zkReLU (points given).

Everything is checked by verifiers written here in Python integers (independent of oracle.c): the
round identities of Protocol 2/3's plain form (g(0) + g(1) = c), the transcript-derived
weights, the verifier-side finals P~ and Wy~ recomputed from the maps and points, the stack's output
claim against its brute-force MLE, and App. A's final identity.
"""
import random

import numpy as np
import pytest

from synth.prng import uniform_range

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def beta_bits(u, b):
    e = 1
    for t, x in enumerate(u):
        e = e * (x if (b >> t) & 1 else 1 - x) % P
    return e


def beta(u, v):
    e = 1
    for a, b in zip(u, v):
        e = e * (a * b + (1 - a) * (1 - b)) % P
    return e


def mle(vals, pt):
    return sum(int(v) * beta_bits(pt, x) for x, v in enumerate(vals)) % P


def lagrange(ev, x):
    K = len(ev) - 1
    tot = 0
    for i in range(K + 1):
        num, den = 1, 1
        for j in range(K + 1):
            if j != i:
                num, den = num * (x - j) % P, den * (i - j) % P
        tot += ev[i] * num * pow(den, -1, P)
    return tot % P


def rounds_ok(claim, msgs, r):
    """Plain-form round identities; returns the final running claim or None."""
    c = claim
    for ev, x in zip(msgs, r):
        if (ev[0] + ev[1]) % P != c:
            return None
        c = lagrange(ev, x)
    return c


def view_claim(X, mp, u, v):
    """X_k~(v, u) = sum_j beta(u, j) X_{map[j]}~(v) (an empty slot is an all-zero slice)."""
    return sum(beta_bits(u, j) * mle(X[i], v) for j, i in enumerate(mp) if i >= 0) % P


def make_claims(rng, X, specs):
    N, D = X.shape
    d = D.bit_length() - 1
    out = []
    for nk, fill in specs:
        slots = 1 << nk
        pick = rng.sample(range(N), min(fill, slots, N))
        mp = pick + [-1] * (slots - len(pick))
        rng.shuffle(mp)
        u = [rng.randrange(P) for _ in range(nk)]
        v = [rng.randrange(P) for _ in range(d)]
        out.append(dict(map=mp, u=u, v=v, c=view_claim(X, mp, u, v)))
    return out


def verify_merge(O, seed, X, claims, res):
    """D25 verifier in Python integers; returns (point, claim) or raises AssertionError."""
    N, D = X.shape
    n, d = N.bit_length() - 1, D.bit_length() - 1
    K = len(claims)
    kap = (K - 1).bit_length()
    tr = O.Transcript(seed)
    hdr = [n, d, K] + [len(c["map"]).bit_length() - 1 for c in claims]
    tr.absorb("cm/hdr", b"".join(x.to_bytes(4, "little") for x in hdr))
    tr.absorb("cm/claims", O.to_bytes([c["c"] for c in claims]))
    rho = tr.challenges("cm/rho", K)
    assert rho == res["rho"]
    cA = sum(r * c["c"] for r, c in zip(rho, claims)) % P
    A = res["A"]
    c = rounds_ok(cA, A["msgs"], A["r"])
    assert c is not None, "phase A round identity"
    assert c == A["finals"][0] * A["finals"][1] % P, "phase A final product"
    ri, rk = A["r"][:n], A["r"][n:]
    Pt = 0
    for k, cl in enumerate(claims):
        s = sum(beta_bits(cl["u"], j) * beta_bits(ri, i) for j, i in enumerate(cl["map"]) if i >= 0)
        Pt += beta_bits(rk, k) * rho[k] * s
    assert A["finals"][0] == Pt % P, "P~ final"
    B = res["B"]
    c = rounds_ok(A["finals"][1], B["msgs"], B["r"])
    assert c is not None, "phase B round identity"
    assert c == B["finals"][0] * B["finals"][1] % P, "phase B final product"
    Wy = sum(beta_bits(rk, k) * beta(cl["v"], B["r"]) for k, cl in enumerate(claims)) % P
    assert B["finals"][0] == Wy, "Wy~ final"
    return B["r"] + ri, B["finals"][1]


@pytest.mark.parametrize("n,d,specs", [(3, 4, [(3, 8), (2, 3), (3, 5)]), (2, 3, [(2, 4)]), (4, 2, [(4, 16), (4, 10)]),
                                       (0, 5, [(0, 1), (0, 1)]), (3, 1, [(3, 7), (1, 2), (2, 4), (0, 1), (3, 8)])])
def test_claim_merge_single_claim_equals_brute_force(oracle_lib, n, d, specs):
    O = oracle_lib
    rng = random.Random(n * 100 + d)
    X = uniform_range(7, n * 10 + d, (1 << n, 1 << d), -(1 << 31), 1 << 31)
    claims = make_claims(rng, X, specs)
    seed = bytes([n, d]) * 16
    res = O.claim_merge_prove(O.Transcript(seed), X, claims)
    pt, cl = verify_merge(O, seed, X, claims, res)
    assert pt == res["point"] and cl == res["claim"]
    assert cl == mle(X.reshape(-1), pt)                          # the one claim left on the stack


def test_claim_merge_rejects_a_false_claim(oracle_lib):
    O = oracle_lib
    rng = random.Random(3)
    X = uniform_range(7, 99, (8, 16), -(1 << 15), 1 << 15)
    for k in range(3):
        claims = make_claims(rng, X, [(3, 8), (2, 4), (3, 6)])
        claims[k]["c"] = (claims[k]["c"] + 1) % P
        res = O.claim_merge_prove(O.Transcript(bytes(32)), X, claims)
        with pytest.raises(AssertionError):
            verify_merge(O, bytes(32), X, claims, res)
    # a wrong map (the verifier's view of which slice a slot holds) is caught by the P~ final
    claims = make_claims(rng, X, [(3, 8), (2, 4)])
    res = O.claim_merge_prove(O.Transcript(bytes(32)), X, claims)
    claims[1]["map"] = claims[1]["map"][::-1]
    with pytest.raises(AssertionError):
        verify_merge(O, bytes(32), X, claims, res)


def test_claim_merge_special_case_is_reindex(oracle_lib):
    """With every inner point equal (the paper's shared u), phase A's claim on the k-combination
    is sum_k beta(r_k, k) X~(u, r_i) = X~(u, r_i): the re-indexing sumcheck's output (D20) at the same
    slice point — checked through the brute-force MLE."""
    O = oracle_lib
    rng = random.Random(11)
    X = uniform_range(7, 55, (8, 8), -(1 << 20), 1 << 20)
    claims = make_claims(rng, X, [(3, 8), (3, 6)])
    v = claims[0]["v"]
    for c in claims:
        c["v"] = v
        c["c"] = view_claim(X, c["map"], c["u"], v)
    res = O.claim_merge_prove(O.Transcript(bytes(32)), X, claims)
    ri = res["A"]["r"][:3]
    assert res["A"]["finals"][1] == mle(X.reshape(-1), v + ri)
    verify_merge(O, bytes(32), X, claims, res)


# ---------------------------------------------------------------- the chained zkReLU (points given)
def relu_final_identity(Z, GA, Q, R, pts, res):
    """App. A's final check at the final point (w over the j bits, v over the i bits), with the verifier's
    own beta, s, s' evaluations."""
    D = len(Z)
    logD = D.bit_length() - 1
    QR = Q + R
    logB = (QR - 1).bit_length()
    B = 1 << logB
    s = [1 << j for j in range(QR - 1)] + [-(1 << (QR - 1))] + [0] * (B - QR)
    sp = [0] * (R - 1) + [1] + [1 << k for k in range(Q - 1)] + [-(1 << (Q - 1))] + [0] * (B - QR)
    x = res["point"]
    w, v = x[:logB], x[logB:]
    sw, spw = mle([t % P for t in s], w), mle([t % P for t in sp], w)
    f0, f1, f2 = res["finals"]
    r, rp, ub = res["r"], res["rp"], res["ubin"]
    eb = beta(ub, w + v)
    uZ, uA, uGA, uGZ = pts
    val = (r * r * beta(uZ, v) * f0 * sw + r * beta(uA, v) * (1 - f2) * f0 * spw + eb * (f0 * f0 - f0)
           + rp * (r * r * beta(uGA, v) * f1 * sw + r * beta(uGZ, v) * (1 - f2) * f1 * spw + eb * (f1 * f1 - f1)))
    # the finals against the brute-force MLEs of the bit tables
    a0 = [((int(Z[i]) & 0xFFFFFFFF) >> j) & 1 if j < QR else 0 for i in range(D) for j in range(B)]
    a1 = [((int(GA[i]) & 0xFFFFFFFF) >> j) & 1 if j < QR else 0 for i in range(D) for j in range(B)]
    sg = [((int(Z[i]) & 0xFFFFFFFF) >> (QR - 1)) & 1 for i in range(D)]
    assert f0 == mle(a0, x) and f1 == mle(a1, x) and f2 == mle(sg, v)
    return val % P


@pytest.mark.parametrize("Q,R,logD", [(4, 2, 3), (16, 16, 4)])
def test_chained_relu_given_points(oracle_lib, Q, R, logD):
    O = oracle_lib
    rng = random.Random(logD)
    half = 1 << (Q + R - 1)
    Z = uniform_range(9, 61, (1 << logD,), -half, half)
    GA = uniform_range(9, 62, (1 << logD,), -half, half)
    pts = [[rng.randrange(P) for _ in range(logD)] for _ in range(4)]
    res = O.relu_prove(O.Transcript(bytes(32)), Z, GA, Q, R, points=pts)
    t = O.relu_tables(Z, GA, Q, R)
    c = res["claims"]                                     # the claims at the GIVEN points (Lemma 1 tensors)
    assert c == [mle(Z, pts[0]), mle(t["A"], pts[1]), mle(GA, pts[2]), mle(t["GZ"], pts[3])]
    # nothing drawn for the points: r, r', u_bin follow "relu/hdr" and "relu/claims" directly
    tr = O.Transcript(bytes(32))
    tr.absorb("relu/hdr", b"".join(int(x).to_bytes(4, "little") for x in (logD, Q, R)))
    tr.absorb("relu/claims", O.to_bytes(c))
    assert tr.challenges("relu/r", 1)[0] == res["r"] and tr.challenges("relu/rp", 1)[0] == res["rp"]
    r, rp = res["r"], res["rp"]
    claim = (r * r * c[0] + r * c[1] + rp * (r * r * c[2] + r * c[3])) % P
    fin = rounds_ok(claim, res["msgs"], res["point"])
    assert fin is not None
    assert fin == relu_final_identity(Z, GA, Q, R, pts, res)
