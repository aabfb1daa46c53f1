"""Exhaustive pins of the oracle's product sumcheck on 2-4 variable inputs (-m "not gpu").

North star: "checked exhaustively on 2-4-variable inputs"; SURVEY.md §8(c) pin table.  Every case
is checked by a verifier written here in Python integers, independent of oracle.c:

* the claim equals the brute-force sum  sum_x beta(w, x_{<n_eq}) prod_k T_k(x)   (Eq. (5));
* round identities: (1 - w_t) f_t(0) + w_t f_t(1) = c_t for t < n_eq (Protocol 3, P:L513, L520,
  the beta(w_t, .) factor and the prefix divided out, D4), g_t(0) + g_t(1) = c_t otherwise
  (Protocol 2); c_{t+1} = the degree-K interpolant of the message at r_t;
* final: c_m = prod_k finals_k and finals_k = T_k~(r) by brute-force MLE of the unfolded table
  (P:L147).

Cases (VERDICT r1 "next" item 1):
* m = 2, K = 2, entries in {0, 1, 2, p-1}: all 256 x 256 (A, B) pairs, each at n_eq = 0, 1 and 2;
* m = 3, K = 2, entries in {0, 1}: all 256 x 256 pairs, n_eq cycling 0..3;
* m = 4, K = 1, entries in {0, 1}: all 2^16 tables, n_eq cycling 0..4.
The work is spread over a process pool (the oracle runs single-threaded per call).
"""
import itertools
import multiprocessing as mp
import os

import pytest

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
# fixed eq points (any field elements work; chosen to have no special structure)
W = [0x1234567890ABCDEF1234567890ABCDEF % P, (P - 7) % P, 0xDEADBEEF, 0x5A5A5A5A5A5A5A5A5A5A5A5A5A5A5A5A]


def _lagrange(ev, x):
    """The degree-len(ev)-1 polynomial through (X, ev[X]), X = 0..K, evaluated at x."""
    K = len(ev) - 1
    tot = 0
    for i in range(K + 1):
        num, den = 1, 1
        for j in range(K + 1):
            if j != i:
                num = num * (x - j) % P
                den = den * (i - j) % P
        tot += ev[i] * num * pow(den, -1, P)
    return tot % P


def _beta_bits(w, x, n):
    e = 1
    for t in range(n):
        e = e * (w[t] if (x >> t) & 1 else 1 - w[t]) % P
    return e


def _mle(tab, pt):
    return sum(tab[x] * _beta_bits(pt, x, len(pt)) for x in range(len(tab))) % P


def _check(m, n_eq, tables, res):
    """0 = the oracle's proof satisfies every identity; else a short reason string."""
    w = W[:n_eq]
    K = len(tables)
    want = 0
    for x in range(1 << m):
        p = _beta_bits(w, x, n_eq)
        for tb in tables:
            p = p * tb[x] % P
        want += p
    if res["claim"] != want % P:
        return "claim"
    c = res["claim"]
    for t in range(m):
        ev = res["msgs"][t]
        if len(ev) != K + 1:
            return "len"
        lhs = ((1 - w[t]) * ev[0] + w[t] * ev[1]) % P if t < n_eq else (ev[0] + ev[1]) % P
        if lhs != c:
            return f"round {t}"
        c = _lagrange(ev, res["r"][t])
    prod = 1
    for f in res["finals"]:
        prod = prod * f % P
    if prod != c:
        return "final product"
    for k, tb in enumerate(tables):
        if res["finals"][k] != _mle(tb, res["r"]):
            return f"final {k}"
    return 0


def _work(args):
    m, K, vals, chunk, n_eq_mode = args
    import oracle as O
    O.set_threads(1)
    bad = []
    n = 0
    tabs = list(itertools.product(vals, repeat=1 << m))
    for ia in chunk:
        A = list(tabs[ia])
        others = tabs if K == 2 else [None]
        for ib, Bt in enumerate(others):
            tables = [A] if K == 1 else [A, list(Bt)]
            eqs = range(m + 1) if n_eq_mode == "all" else [(ia + ib) % (m + 1)]
            for n_eq in eqs:
                res = O.sumcheck_prove(O.Transcript(bytes([m, K, n_eq]) + bytes(29)), m, n_eq, tables, W[:n_eq])
                why = _check(m, n_eq, tables, res)
                n += 1
                if why:
                    bad.append((ia, ib, n_eq, why))
                    if len(bad) > 5:
                        return n, bad
    return n, bad


def _run(m, K, vals, n_eq_mode):
    import oracle
    oracle.build()
    ntab = len(vals) ** (1 << m)
    nproc = max(1, min(16, os.cpu_count() or 1))
    chunks = [list(range(i, ntab, nproc * 4)) for i in range(nproc * 4)]
    with mp.get_context("spawn").Pool(nproc) as pool:
        out = pool.map(_work, [(m, K, vals, c, n_eq_mode) for c in chunks])
    total = sum(o[0] for o in out)
    bad = [b for o in out for b in o[1]]
    return total, bad


@pytest.mark.slow
def test_exhaustive_m2_k2_all_pairs_all_neq():
    total, bad = _run(2, 2, [0, 1, 2, P - 1], "all")
    assert not bad, bad[:5]
    assert total == 256 * 256 * 3


@pytest.mark.slow
def test_exhaustive_m3_k2_binary_all_pairs():
    total, bad = _run(3, 2, [0, 1], "cycle")
    assert not bad, bad[:5]
    assert total == 256 * 256


@pytest.mark.slow
def test_exhaustive_m4_k1_binary_all_tables():
    total, bad = _run(4, 1, [0, 1], "cycle")
    assert not bad, bad[:5]
    assert total == 1 << 16


def test_python_checker_catches_mistakes(oracle_lib):
    """The checker above is itself pinned: a dropped term, a wrong sign, a transposed operand or a
    wrong final each make it fail."""
    O = oracle_lib
    O.set_threads(1)
    A, B = [3, 1, 4, 1, 5, 9, 2, 6], [2, 7, 1, 8, 2, 8, 1, 8]
    for n_eq in range(4):
        res = O.sumcheck_prove(O.Transcript(bytes(32)), 3, n_eq, [A, B], W[:n_eq])
        assert _check(3, n_eq, [A, B], res) == 0
        bad = dict(res, msgs=[list(r) for r in res["msgs"]])
        bad["msgs"][1][2] = (bad["msgs"][1][2] + 1) % P                 # one evaluation off
        assert _check(3, n_eq, [A, B], bad) != 0
        bad = dict(res, finals=[res["finals"][1], res["finals"][0]])    # operands swapped
        assert _check(3, n_eq, [A, B], bad) != 0 or res["finals"][0] == res["finals"][1]
        bad = dict(res, claim=(res["claim"] + 1) % P)
        assert _check(3, n_eq, [A, B], bad) != 0
        assert _check(3, n_eq, [A, [-v % P for v in B]], res) != 0      # sign of an operand
