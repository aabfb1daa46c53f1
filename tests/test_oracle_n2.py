"""Pins for the oracle's SURVEY §8(f) N2 step (-m "not gpu"): Protocol 2's zero form for the aggregated
Hadamard product (Eq. tensor-op-aggr, Protocol 2 P:L476-502; D22).

The verifier is written here from Protocol 2 (g_t = beta(w_t, .) f_t, g_0(0) + g_0(1) = 0,
g_t(0) + g_t(1) = f_{t-1}(v_{t-1}), the last claim against Y~ - A~ B~ at the final point) with every
multilinear extension evaluated by Python-int brute force; tampering with one entry of Y must break
the first identity.
"""
import numpy as np
import pytest

from synth.prng import fs_seed, uniform_range

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def mle(vals, point):
    acc = 0
    for b, v in enumerate(vals):
        w = 1
        for t, x in enumerate(point):
            w = w * (x if (b >> t) & 1 else 1 - x) % P
        acc = (acc + int(v) * w) % P
    return acc


def lagrange3(e, x):
    inv2 = pow(2, P - 2, P)
    return (e[0] * (x - 1) * (x - 2) * inv2 - e[1] * x * (x - 2) + e[2] * x * (x - 1) * inv2) % P


def verify(O, seed, m, res, Y, A, B):
    """Protocol 2 verifier; returns 0 = accept, t + 1 = the failing round, -1 = the final check."""
    tr = O.Transcript(seed)
    tr.absorb("hd/hdr", m.to_bytes(4, "little"))
    w = tr.challenges("hd/w", m)
    assert w == res["w"]
    c = 0
    for t, e in enumerate(res["msgs"]):
        if ((1 - w[t]) * e[0] + w[t] * e[1]) % P != c:
            return t + 1
        tr.absorb("sc/msg", O.to_bytes(e))
        r = tr.challenges("sc/r", 1)[0]
        assert r == res["r"][t]
        c = lagrange3(e, r)
    y, a, b = (mle(list(T), res["r"]) for T in (Y, A, B))
    if res["finals"] != [y, a, b] or c != (y - a * b) % P:
        return -1
    return 0


def test_zero_form_honest_hadamard_accepted(oracle_lib):
    O = oracle_lib
    for m in (1, 2, 3, 5, 7):
        A = uniform_range(31, m, (1 << m,), -(1 << 15), 1 << 15)
        B = uniform_range(31, m + 40, (1 << m,), -(1 << 15), 1 << 15)
        Y = (A.astype(np.int64) * B).astype(np.int32)
        seed = fs_seed(f"hd-{m}")
        res = O.zero_sumcheck_prove(O.Transcript(seed), Y, A, B)
        assert verify(O, seed, m, res, Y, A, B) == 0
        # the statement itself: sum_x beta(w, x) (Y - A B) = 0, and f_0 folds to it
        w = res["w"]
        total = sum(mle([1 if i == x else 0 for i in range(1 << m)], w) * (int(Y[x]) - int(A[x]) * int(B[x]))
                    for x in range(1 << m)) % P
        assert total == 0


def test_zero_form_rejects_a_wrong_product(oracle_lib):
    O = oracle_lib
    m = 6
    A = uniform_range(32, 1, (1 << m,), -(1 << 15), 1 << 15)
    B = uniform_range(32, 2, (1 << m,), -(1 << 15), 1 << 15)
    for pos in (0, 17, 63):
        Y = (A.astype(np.int64) * B).astype(np.int32)
        Y[pos] += 1
        seed = fs_seed(f"hd-bad-{pos}")
        res = O.zero_sumcheck_prove(O.Transcript(seed), Y, A, B)
        assert verify(O, seed, m, res, Y, A, B) == 1


# ---------------------------------------------------------------- the loss-gradient family (D24)
def test_loss_grad_claims_brute_force_and_linearity(oracle_lib):
    """Eq. (fcnn-GZ-last): the three claims are the brute-force MLEs at the transcript's u
    (drawn "lg/u" after "lg/hdr"), G_Z~(u) = Z~(u) - Y~(u) for G_Z = Z - Y, and a changed entry of G_Z
    breaks the identity (its MLE moves by beta(u, x) != 0)."""
    O = oracle_lib
    for m in (1, 3, 6):
        Z = uniform_range(33, m, (1 << m,), -(1 << 20), 1 << 20)
        Y = uniform_range(33, m + 20, (1 << m,), -(1 << 20), 1 << 20)
        G = (Z.astype(np.int64) - Y).astype(np.int32)
        seed = fs_seed(f"lg-{m}")
        res = O.loss_grad_prove(O.Transcript(seed), G, Z, Y)
        T = O.Transcript(seed)
        T.absorb("lg/hdr", m.to_bytes(4, "little"))
        u = T.challenges("lg/u", m)
        assert res["u"] == u
        g, z, y = res["claims"]
        assert [g, z, y] == [mle(list(G), u), mle(list(Z), u), mle(list(Y), u)]
        assert g == (z - y) % P
        Gb = G.copy()
        Gb[(1 << m) - 1] += 1
        gb = O.loss_grad_prove(O.Transcript(seed), Gb, Z, Y)["claims"][0]
        assert gb != (z - y) % P


# ---------------------------------------------------------------- the top-layer rescale (D26)
def _beta_pt(u, v):
    e = 1
    for a, b in zip(u, v):
        e = e * (a * b + (1 - a) * (1 - b)) % P
    return e


def _lag(ev, x):
    K = len(ev) - 1
    tot = 0
    for i in range(K + 1):
        num, den = 1, 1
        for j in range(K + 1):
            if j != i:
                num, den = num * (x - j) % P, den * (i - j) % P
        tot += ev[i] * num * pow(den, -1, P)
    return tot % P


def _rescale_check(Z, Q, R, pts, res, claims=None):
    """D26 verifier in Python integers: A's and B's round identities, A's weight final recomputed, B's
    second final = first - 1, both aux finals = brute-force MLEs of the bits of Z."""
    D = len(Z)
    logD = D.bit_length() - 1
    QR = Q + R
    logB = (QR - 1).bit_length()
    Bc = 1 << logB
    cz, cp = res["claims"] if claims is None else claims
    r = res["r"]
    c = (r * cz + cp) % P
    A = res["A"]
    for ev, x in zip(A["msgs"], A["r"]):
        assert (ev[0] + ev[1]) % P == c, "A round"
        c = _lag(ev, x)
    assert c == A["finals"][0] * A["finals"][1] % P
    rj, ri = A["r"][:logB], A["r"][logB:]
    s = [1 << j for j in range(QR - 1)] + [-(1 << (QR - 1))] + [0] * (Bc - QR)
    sp = [0] * (R - 1) + [1] + [1 << k for k in range(Q - 1)] + [-(1 << (Q - 1))] + [0] * (Bc - QR)
    sw, spw = mle([x % P for x in s], rj), mle([x % P for x in sp], rj)
    assert A["finals"][0] == (r * _beta_pt(pts[0], ri) * sw + _beta_pt(pts[1], ri) * spw) % P, "W final"
    bits = [((int(z) & 0xFFFFFFFF) >> j) & 1 if j < QR else 0 for z in Z for j in range(Bc)]
    assert A["finals"][1] == mle(bits, A["r"])
    B = res["B"]
    c, w = 0, res["w"]
    for t, (ev, x) in enumerate(zip(B["msgs"], B["r"])):
        assert ((1 - w[t]) * ev[0] + w[t] * ev[1]) % P == c, "B round"
        c = _lag(ev, x)
    assert c == B["finals"][0] * B["finals"][1] % P
    assert B["finals"][1] == (B["finals"][0] - 1) % P
    assert B["finals"][0] == mle(bits, B["r"])


@pytest.mark.parametrize("Q,R,logD", [(4, 2, 3), (16, 16, 4), (8, 8, 5)])
def test_rescale_claims_identities_and_finals(oracle_lib, Q, R, logD):
    import random
    O = oracle_lib
    rng = random.Random(logD * 7 + Q)
    half = 1 << (Q + R - 1)
    Z = uniform_range(45, logD, (1 << logD,), -half, half)
    Z[0], Z[1] = half - 1, -half                    # both ends of the range (the D11 edge included)
    pts = [[rng.randrange(P) for _ in range(logD)] for _ in range(2)]
    res = O.rescale_prove(O.Transcript(bytes(32)), Z, Q, R, pts)
    Zp = [(int(z) + (1 << (R - 1))) >> R for z in Z]   # round(Z / 2^R), half-up (D9)
    assert res["claims"] == [mle(Z, pts[0]), mle(Zp, pts[1])]
    _rescale_check(Z, Q, R, pts, res)


def test_rescale_rejects_other_rounding(oracle_lib):
    """A claim on round-toward-zero (or floor) instead of the half-up Z' of D9 fails A's first round."""
    import random
    O = oracle_lib
    rng = random.Random(9)
    Q, R, logD = 4, 2, 4
    Z = np.array([-7, -6, -5, -3, -2, -1, 0, 1, 2, 3, 5, 6, 7, 9, 10, 13], dtype=np.int32)
    pts = [[rng.randrange(P) for _ in range(logD)] for _ in range(2)]
    res = O.rescale_prove(O.Transcript(bytes(32)), Z, Q, R, pts)
    trunc = [int(np.trunc(int(z) / 4)) for z in Z]
    floor_ = [int(z) >> R for z in Z]
    for other in (trunc, floor_):
        with pytest.raises(AssertionError):
            _rescale_check(Z, Q, R, pts, res, claims=[res["claims"][0], mle(other, pts[1])])
