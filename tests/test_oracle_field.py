"""Pins for the oracle's field arithmetic, SHA-256 and transcript (-m "not gpu").

Each check compares the C oracle with something other than itself: Python
integers (the definition of Z/pZ), the BLS12-381 parameter identity, RFC 7693
BLAKE2s vectors (RFC 7693), hashlib, and SPEC's worked examples.
"""
import hashlib
import random

import pytest

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
BLS_X = -0xD201000000010000


def _is_probable_prime(n, bases=(2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)):
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in bases:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def test_modulus_is_bls12_381_scalar_field(oracle_lib):
    # D1: the BLS12-381 scalar field r = x^4 - x^2 + 1 for the curve parameter x
    assert P == BLS_X ** 4 - BLS_X ** 2 + 1
    assert P.bit_length() == 255 and _is_probable_prime(P)
    assert (P - 1) % (1 << 32) == 0 and ((P - 1) >> 32) % 2 == 1     # 2-adicity 32
    assert oracle_lib.P == P


def test_pinv(oracle_lib):
    assert (P * oracle_lib.pinv()) % (1 << 64) == (1 << 64) - 1


def test_field_ops_vs_python_ints(oracle_lib):
    rng = random.Random(7)
    edges = [0, 1, 2, P - 1, P - 2, (1 << 256) % P, (1 << 255) % P, (1 << 64) - 1, 1 << 128]
    vals = edges + [rng.randrange(P) for _ in range(300)]
    for a in vals:
        for b in rng.sample(vals, 6) + [0, 1, P - 1]:
            assert oracle_lib.fr_op("add", a, b) == (a + b) % P
            assert oracle_lib.fr_op("sub", a, b) == (a - b) % P
            assert oracle_lib.fr_op("mul", a, b) == a * b % P
        assert oracle_lib.fr_op("neg", a) == (-a) % P
        if a:
            assert oracle_lib.fr_op("inv", a) * a % P == 1


def test_noncanonical_rejected(oracle_lib):
    for bad in (P, P + 1, (1 << 256) - 1):
        with pytest.raises(ValueError):
            oracle_lib.fr_op("add", bad, 0)


def test_embed_spec_examples(oracle_lib):
    # embed(0) = 0, embed(-1) = p - 1; embed(3)*embed(-2) lifts to -6
    e = oracle_lib.embed([0, -1, 3, -2, -(1 << 31), (1 << 31) - 1])
    assert e[0] == 0 and e[1] == P - 1
    assert oracle_lib.fr_op("mul", e[2], e[3]) == P - 6
    assert e[4] == P - (1 << 31) and e[5] == (1 << 31) - 1


# RFC 7693 Appendix B: BLAKE2s-256("abc"); the empty message (BLAKE2 reference test vectors)
B2S = [
    (b"abc", "508c5e8c327c14e2e1a72ba34eeb452f37458b209ed63a294d999b4c86675982"),
    (b"", "69217a3079908094e11121d042354a7c1f55b6482ca1a51e1b250dfd1ed0eef9"),
]


@pytest.mark.parametrize("msg,hexd", B2S)
def test_blake2s_rfc7693(oracle_lib, msg, hexd):
    assert oracle_lib.blake2s(msg).hex() == hexd


def test_blake2s_vs_hashlib(oracle_lib):
    """Every length around the 64-byte block boundaries (the final block is never empty-padded)."""
    rng = random.Random(3)
    for n in list(range(0, 200)) + [1000, 4096, 4097]:
        m = bytes(rng.randrange(256) for _ in range(n))
        assert oracle_lib.blake2s(m) == hashlib.blake2s(m).digest()


def _ref_transcript(seed, ops):
    """DESIGN.md D3 written with hashlib (independent BLAKE2s + big-int reduction)."""
    H = lambda b: hashlib.blake2s(b).digest()
    st = H(b"zkdl-b200/v1/init" + seed)
    outs = []
    for op in ops:
        if op[0] == "absorb":
            tag, msg = op[1].encode(), op[2]
            st = H(st + b"\x01" + bytes([len(tag)]) + tag + len(msg).to_bytes(8, "big") + msg)
        else:
            tag = op[1].encode()
            for _ in range(op[2]):
                st = H(st + b"\x02" + bytes([len(tag)]) + tag)
                outs.append(int.from_bytes(H(st + b"\x00") + H(st + b"\x01"), "little") % P)
    return st, outs


def test_transcript_matches_definition(oracle_lib):
    seed = hashlib.sha256(b"zkdl-b200/fs-seed/test").digest()
    ops = [("absorb", "mm/hdr", b"\x01\x00\x00\x00" * 4), ("ch", "mm/w", 3), ("absorb", "sc/msg", bytes(96)),
           ("ch", "sc/r", 1), ("absorb", "x", b""), ("ch", "y", 2)]
    tr = oracle_lib.Transcript(seed)
    got = []
    for op in ops:
        if op[0] == "absorb":
            tr.absorb(op[1], op[2])
        else:
            got += tr.challenges(op[1], op[2])
    st, want = _ref_transcript(seed, ops)
    assert got == want and tr.state() == st
    assert all(0 <= x < P for x in got)


def test_transcript_sensitivity(oracle_lib):
    # any byte change in an absorbed message changes every later challenge
    a, b = oracle_lib.Transcript(bytes(32)), oracle_lib.Transcript(bytes(32))
    a.absorb("t", b"hello")
    b.absorb("t", b"hellp")
    assert a.challenges("c", 4) != b.challenges("c", 4)
    # framing: absorb(a||b) != absorb(a); absorb(b)
    a, b = oracle_lib.Transcript(bytes(32)), oracle_lib.Transcript(bytes(32))
    a.absorb("t", b"ab")
    b.absorb("t", b"a")
    b.absorb("t", b"b")
    assert a.state() != b.state()
