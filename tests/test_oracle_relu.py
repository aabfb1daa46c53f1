"""Pins for the oracle's zkReLU (Sec. 3, App. A, Lemma 1) (-m "not gpu").

Pinned against: SPEC's worked examples, Lemma 1
 exhaustively at Q=4 R=2 via the bit relations of Eqs. (aux-*)
(P:L188-205), the D11 top edge, the six-statement combination's claim equal to
its brute-force double sum, verifier acceptance, and tampering.
"""
import random

import numpy as np
import pytest

from synth.prng import uniform_range

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def bits(v, n):
    return [(v >> j) & 1 for j in range(n)]


def s_vec(B):
    return [1 << j for j in range(B - 1)] + [-(1 << (B - 1))]


def test_round_rescale_spec(oracle_lib):
    O = oracle_lib
    t = O.relu_tables(np.array([3 * 65536 + 5], np.int32), np.array([0], np.int32), 16, 16)
    assert t["Zp"][0] == 3 and t["RZ"][0] == 5
    t = O.relu_tables(np.array([-1, 6], np.int32), np.array([0, 0], np.int32), 4, 2)
    assert list(t["Zp"]) == [0, 2] and list(t["RZ"]) == [-1, -2]


def test_spec_zkrelu_example(oracle_lib):
    # Q=4, R=2, Z = -3 -> bits (1,0,1,1,1,1), Z' = -1, R_Z = 1, A = 0
    O = oracle_lib
    t = O.relu_tables(np.array([-3], np.int32), np.array([0], np.int32), 4, 2)
    assert bits(-3 & 63, 6) == [1, 0, 1, 1, 1, 1]
    assert t["Zp"][0] == -1 and t["RZ"][0] == 1 and t["A"][0] == 0 and t["sign"][0] == 1


def test_lemma1_exhaustive_q4_r2(oracle_lib):
    """For every (Z, G_A) in [-32, 32)^2 the bit relations (aux-Z, aux-GA, aux-A, aux-GZ) hold with
    the Lemma-1 values A = round(1{Z>=0} Z / 2^R), G_Z = round(1{Z>=0} G_A / 2^R)."""
    O = oracle_lib
    Q, R = 4, 2
    QR = Q + R
    zs = np.repeat(np.arange(-32, 32, dtype=np.int32), 64)
    gs = np.tile(np.arange(-32, 32, dtype=np.int32), 64)
    t = O.relu_tables(zs, gs, Q, R)
    sQR, sQ, sR = s_vec(QR), s_vec(Q), s_vec(R)
    for i in range(zs.size):
        z, g = int(zs[i]), int(gs[i])
        a0, a1 = bits(z & 63, QR), bits(g & 63, QR)
        assert sum(x * w for x, w in zip(a0, sQR)) == z                                  # aux-Z
        assert sum(x * w for x, w in zip(a1, sQR)) == g                                  # aux-GA
        zp = sum(x * w for x, w in zip(a0[R:], sQ)) + a0[R - 1]
        gp = sum(x * w for x, w in zip(a1[R:], sQ)) + a1[R - 1]
        assert sum(x * w for x, w in zip(a0[:R], sR)) == z - (zp << R)                # R_Z
        sig = a0[QR - 1]
        assert sig == (z < 0)
        assert t["A"][i] == (1 - sig) * zp                                               # aux-A
        assert t["GZ"][i] == (1 - sig) * gp                                              # aux-GZ
        assert t["Zp"][i] == zp and t["GAp"][i] == gp
        assert -(1 << (R - 1)) <= t["RZ"][i] < (1 << (R - 1))


def test_top_edge_d11(oracle_lib):
    # Z >= 2^{Q+R-1} - 2^{R-1} rounds to Z' = 2^{Q-1}, outside the Q-bit range; relations still hold
    O = oracle_lib
    t = O.relu_tables(np.array([31], np.int32), np.array([31], np.int32), 4, 2)
    assert t["Zp"][0] == 8 and t["A"][0] == 8 and t["RZ"][0] == -1


def test_range_violation(oracle_lib):
    O = oracle_lib
    with pytest.raises(ValueError):
        O.relu_tables(np.array([32], np.int32), np.array([0], np.int32), 4, 2)


def _six_statement_sum(Z, GA, Q, R, ch):
    """Brute-force double sum of App. A's six statements with weights r^2, r, 1, r'r^2, r'r, r'."""
    D = len(Z)
    logD = D.bit_length() - 1
    QR = Q + R
    logB = (QR - 1).bit_length()
    B = 1 << logB
    r, rp, ub = ch["r"], ch["rp"], ch["ubin"]
    uZ, uA, uGA, uGZ = ch["uZ"], ch["uA"], ch["uGA"], ch["uGZ"]

    def eq(u, b):
        e = 1
        for t, x in enumerate(u):
            e = e * (x if (b >> t) & 1 else 1 - x) % P
        return e
    s = [1 << j for j in range(QR - 1)] + [-(1 << (QR - 1))] + [0] * (B - QR)
    sp = [0] * (R - 1) + [1] + [1 << k for k in range(Q - 1)] + [-(1 << (Q - 1))] + [0] * (B - QR)
    tot = 0
    for i in range(D):
        z, g = int(Z[i]) & 0xFFFFFFFF, int(GA[i]) & 0xFFFFFFFF
        sig = (z >> (QR - 1)) & 1
        for j in range(B):
            a0 = (z >> j) & 1 if j < QR else 0
            a1 = (g >> j) & 1 if j < QR else 0
            eb = eq(ub, i * B + j)
            tot += r * r * eq(uZ, i) * a0 * s[j] + r * eq(uA, i) * (1 - sig) * a0 * sp[j] + eb * (a0 * a0 - a0)
            tot += rp * (r * r * eq(uGA, i) * a1 * s[j] + r * eq(uGZ, i) * (1 - sig) * a1 * sp[j] + eb * (a1 * a1 - a1))
    return tot % P


@pytest.mark.parametrize("Q,R,logD", [(4, 2, 3), (4, 4, 4), (16, 16, 3)])
def test_relu_prove_verify_and_six_statement_identity(oracle_lib, Q, R, logD):
    O = oracle_lib
    half = 1 << (Q + R - 1)
    Z = uniform_range(4, 61, (1 << logD,), -half, half)
    GA = uniform_range(4, 62, (1 << logD,), -half, half)
    seed = bytes([Q, R, logD]) * 10 + b"zz"
    res = O.relu_prove(O.Transcript(seed), Z, GA, Q, R)
    assert O.relu_verify(O.Transcript(seed), Z, GA, Q, R, res["claims"], res["msgs"], res["finals"]) == 0
    # recover the points the transcript drew (same order as the prover)
    tr = O.Transcript(seed)
    tr.absorb("relu/hdr", b"".join(int(x).to_bytes(4, "little") for x in (logD, Q, R)))
    ch = dict(uZ=tr.challenges("relu/uZ", logD), uA=tr.challenges("relu/uA", logD),
              uGA=tr.challenges("relu/uGA", logD), uGZ=tr.challenges("relu/uGZ", logD),
              r=res["r"], rp=res["rp"], ubin=res["ubin"])
    r, rp = res["r"], res["rp"]
    c = res["claims"]
    claim = (r * r * c[0] + r * c[1] + rp * (r * r * c[2] + r * c[3])) % P
    assert _six_statement_sum(Z, GA, Q, R, ch) == claim
    assert (res["msgs"][0][0] + res["msgs"][0][1]) % P == claim
    # claims equal the MLEs of Z, A, G_A, G_Z with A, G_Z from Lemma 1
    t = O.relu_tables(Z, GA, Q, R)
    assert c[0] == O.mle_i32(Z, ch["uZ"]) and c[1] == O.mle_i32(t["A"], ch["uA"])
    assert c[2] == O.mle_i32(GA, ch["uGA"]) and c[3] == O.mle_i32(t["GZ"], ch["uGZ"])


def test_relu_soundness_wrong_activation(oracle_lib):
    """A prover whose A deviates in one entry cannot satisfy the combined statement (Thm. 2)."""
    O = oracle_lib
    Q, R, logD = 4, 2, 3
    Z = uniform_range(5, 71, (8,), -32, 32)
    GA = uniform_range(5, 72, (8,), -32, 32)
    res = O.relu_prove(O.Transcript(bytes(32)), Z, GA, Q, R)
    tr = O.Transcript(bytes(32))
    tr.absorb("relu/hdr", b"".join(int(x).to_bytes(4, "little") for x in (logD, Q, R)))
    ch = dict(uZ=tr.challenges("relu/uZ", logD), uA=tr.challenges("relu/uA", logD),
              uGA=tr.challenges("relu/uGA", logD), uGZ=tr.challenges("relu/uGZ", logD),
              r=res["r"], rp=res["rp"], ubin=res["ubin"])
    t = O.relu_tables(Z, GA, Q, R)
    A_bad = t["A"].copy()
    A_bad[3] += 1
    r, rp = res["r"], res["rp"]
    c = res["claims"]
    bad_claim = (r * r * c[0] + r * O.mle_i32(A_bad, ch["uA"]) + rp * (r * r * c[2] + r * c[3])) % P
    assert _six_statement_sum(Z, GA, Q, R, ch) != bad_claim


def test_relu_tamper_rejected(oracle_lib):
    O = oracle_lib
    rng = random.Random(5)
    Q, R, logD = 4, 4, 4
    Z = uniform_range(6, 81, (16,), -128, 128)
    GA = uniform_range(6, 82, (16,), -128, 128)
    res = O.relu_prove(O.Transcript(bytes(32)), Z, GA, Q, R)
    m = len(res["msgs"])
    for trial in range(60):
        msgs = [list(x) for x in res["msgs"]]
        fin = list(res["finals"])
        cl = list(res["claims"])
        k = trial % 3
        if k == 0:
            t, x = rng.randrange(m), rng.randrange(4)
            msgs[t][x] = (msgs[t][x] + 1 + rng.randrange(P - 1)) % P
        elif k == 1:
            fin[rng.randrange(3)] ^= 1
        else:
            j = rng.randrange(4)
            cl[j] = (cl[j] + 1) % P
        assert O.relu_verify(O.Transcript(bytes(32)), Z, GA, Q, R, cl, msgs, fin) != 0
