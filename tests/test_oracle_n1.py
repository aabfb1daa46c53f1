"""Pins for the oracle's SURVEY §8(f) N1 steps (-m "not gpu"): the re-indexing sumcheck of
Eq. (sc-reindex) (D20) and the zkReLU aux-claim merge (D21).

Pinned against Python-int brute force written from the definitions (multilinear extensions as sums
over the Boolean cube, the views materialised slot by slot, aux as the dense bit tensor), the SPEC
examples of prove_reindex, the sumcheck verifier's round identities, and tampering.
"""
import random

import numpy as np

from synth.prng import fs_seed, uniform_range

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def mle(vals, point):
    """sum_b vals[b] prod_t (point_t if bit t of b else 1 - point_t) mod P (LSB-first, D2)."""
    acc = 0
    for b, v in enumerate(vals):
        if v % P == 0:
            continue
        w = 1
        for t, x in enumerate(point):
            w = w * (x if (b >> t) & 1 else 1 - x) % P
        acc = (acc + v * w) % P
    return acc


def view_rows(X, mp):
    N, D = X.shape
    return np.stack([X[i] if i >= 0 else np.zeros(D, np.int64) for i in mp]).astype(np.int64)


def make_case(rng, n, d, nks, seed):
    X = uniform_range(seed, 1, (1 << n, 1 << d), -(1 << 15), 1 << 15)
    u = [rng.randrange(P) for _ in range(d)]
    views = []
    for nk in nks:
        slots = 1 << nk
        pick = rng.sample(range(1 << n), min(slots, 1 << n))
        mp = pick + [-1] * (slots - len(pick))
        rng.shuffle(mp)
        views.append((mp, [rng.randrange(P) for _ in range(nk)]))
    # c_k = X_k~(u, u_k): the view materialised, its MLE by brute force (point: D bits, then slots)
    claims = [mle([int(v) for v in view_rows(X, mp).reshape(-1)], u + uk) for mp, uk in views]
    return X, u, views, claims


def test_reindex_identity_and_final_claims(oracle_lib):
    O = oracle_lib
    rng = random.Random(5)
    for (n, d, nks) in [(3, 2, [3, 2, 1]), (4, 1, [4, 4]), (2, 3, [0, 1, 2]), (5, 2, [3])]:
        X, u, views, claims = make_case(rng, n, d, nks, 40 + n)
        tr = O.Transcript(fs_seed(f"rx-{n}-{d}"))
        res = O.reindex_prove(tr, X, views, u, claims, want_tables=True)
        rk = res["rk"]
        # Eq. (sc-reindex): sum_k r_k c_k = sum_i C(i) X~(u, i), C and X_u from their definitions
        C = [0] * (1 << n)
        for (mp, uk), r in zip(views, rk):
            for j, i in enumerate(mp):
                if i >= 0:
                    C[i] = (C[i] + r * mle([1 if x == j else 0 for x in range(len(mp))], uk)) % P
        Xu = [mle([int(v) for v in X[i]], u) for i in range(1 << n)]
        assert res["C"] == C and res["Xu"] == Xu
        lhs = sum(r * c for r, c in zip(rk, claims)) % P
        assert res["claim"] == lhs == sum(a * b for a, b in zip(C, Xu)) % P
        # finals: C~(r) and X~(u, r) (the output claim on the stacked tensor)
        assert res["finals"][0] == mle(C, res["r"])
        assert res["finals"][1] == mle([int(v) for v in X.reshape(-1)], u + res["r"])


def test_reindex_spec_examples(oracle_lib):
    O = oracle_lib
    rng = random.Random(6)
    # K = 1, identity permutation -> the output claim is X at (u, r) and C = r_0 beta(u_0, .)
    X = uniform_range(7, 2, (8, 4), -128, 128)
    u, u0 = [rng.randrange(P) for _ in range(2)], [rng.randrange(P) for _ in range(3)]
    c0 = mle([int(v) for v in X.reshape(-1)], u + u0)
    res = O.reindex_prove(O.Transcript(b"\x01" * 32), X, [(list(range(8)), u0)], u, [c0], want_tables=True)
    assert res["C"] == [res["rk"][0] * mle([1 if x == i else 0 for x in range(8)], u0) % P for i in range(8)]
    # X = stack(A, B), X_0 = (B): weight vector (0, r_0 beta((), 0)) = (0, r_0)
    AB = uniform_range(7, 3, (2, 4), -128, 128)
    cB = mle([int(v) for v in AB[1]], u)
    res = O.reindex_prove(O.Transcript(b"\x02" * 32), AB, [([1], [])], u, [cB], want_tables=True)
    assert res["C"] == [0, res["rk"][0]]
    assert res["finals"][1] == mle([int(v) for v in AB.reshape(-1)], u + res["r"])


def test_reindex_verifier_accepts_and_rejects_tampering(oracle_lib):
    O = oracle_lib
    rng = random.Random(7)
    X, u, views, claims = make_case(rng, 4, 2, [3, 4], 77)
    seed = fs_seed("rx-verify")

    def replay(cl):
        tr = O.Transcript(seed)
        hdr = b"".join(v.to_bytes(4, "little") for v in [4, 2, 2, 3, 4])
        tr.absorb("rx/hdr", hdr)
        tr.absorb("rx/claims", O.to_bytes(cl))
        rk = tr.challenges("rx/r", 2)
        return tr, sum(r * c for r, c in zip(rk, cl)) % P

    res = O.reindex_prove(O.Transcript(seed), X, views, u, claims, want_tables=True)
    tr, claim = replay(claims)
    assert claim == res["claim"]
    assert O.sumcheck_verify(tr, 4, 0, 2, [], claim, res["msgs"], res["finals"], tables=[res["C"], res["Xu"]]) == 0
    bad = list(claims)
    bad[1] = (bad[1] + 1) % P                 # an inflated view claim: the first round fails
    res2 = O.reindex_prove(O.Transcript(seed), X, views, u, bad, want_tables=True)
    tr, claim = replay(bad)
    assert O.sumcheck_verify(tr, 4, 0, 2, [], claim, res2["msgs"], res2["finals"]) == 1


def aux_dense(Z, GA, logB, QR):
    """aux[s][i][j] = bit j of the (Q+R)-bit two's-complement word (zero for j >= Q+R, D12),
    flattened with j lowest, then i, then s (D2)."""
    B = 1 << logB
    out = []
    for word in (Z, GA):
        for x in word:
            out += [((int(x) & 0xFFFFFFFF) >> j) & 1 if j < QR else 0 for j in range(B)]
    return out


def test_relu_merge_single_claim(oracle_lib):
    O = oracle_lib
    for (Q, R, logD) in [(4, 2, 3), (16, 16, 2), (8, 8, 4)]:
        half = 1 << (Q + R - 1)
        Z = uniform_range(9, logD + Q, (1 << logD,), -half, half)
        GA = uniform_range(9, logD + R + 50, (1 << logD,), -half, half)
        tr = O.Transcript(fs_seed(f"merge-{Q}-{R}-{logD}"))
        pr = O.relu_prove(tr, Z, GA, Q, R)
        mg = O.relu_merge(tr, Z, GA, Q, R, pr["point"], pr["finals"])
        logB = O.relu_logB(Q, R)
        w, v = pr["point"][:logB], pr["point"][logB:]
        # the three claims are MLEs of the dense aux tensor (Q+R-1 is a Boolean j-point)
        aux = aux_dense(Z, GA, logB, Q + R)
        top = [(Q + R - 1 >> t) & 1 for t in range(logB)]
        f0, f1, f2 = mle(aux, w + v + [0]), mle(aux, w + v + [1]), mle(aux, top + v + [0])
        assert pr["finals"] == [f0, f1, f2]
        rho = mg["rho"]
        assert mg["claim"] == (f0 + rho * f1 + rho * rho * f2) % P
        # the merged claim: aux~ at (r_j, v, r_s), one point
        rj, rs = mg["r"][:logB], mg["r"][logB]
        assert mg["finals"][0] == mle(aux, rj + v + [rs])
        # W~(r) is the verifier's: [s=0](beta(w, r_j) + rho^2 beta(Q+R-1, r_j)) + [s=1] rho beta(w, r_j)
        bw = mle([1 if j == 0 else 0 for j in range(1)], [])   # 1
        ew = mle([mle([1 if x == j else 0 for x in range(1 << logB)], w) for j in range(1 << logB)], rj)
        et = mle([1 if j == Q + R - 1 else 0 for j in range(1 << logB)], rj)
        W = ((1 - rs) * (ew + rho * rho * et) + rs * rho * ew) * bw % P
        assert mg["finals"][1] == W
        assert mg["finals"][0] * mg["finals"][1] % P == interp_last(mg, P)


def interp_last(mg, P):
    """The last round's message evaluated at its challenge (Lagrange through 0, 1, 2)."""
    e, x = mg["msgs"][-1], mg["r"][-1]
    inv2 = pow(2, P - 2, P)
    l0 = (x - 1) * (x - 2) * inv2 % P
    l1 = -x * (x - 2) % P
    l2 = x * (x - 1) * inv2 % P
    return (e[0] * l0 + e[1] * l1 + e[2] * l2) % P
