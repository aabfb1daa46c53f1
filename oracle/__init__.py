"""CPU oracle for the zkDL sumcheck hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
``--impl reference`` arm) may import this package.  The product path
(paper_2307_16273_b200) never imports it and shares no code with it.

The arithmetic lives in oracle.c (plain C, 4x64-bit Montgomery Fr, plain
SHA-256, brute-force eq/MLE, dense sumcheck provers and verifiers); this module
only marshals bytes through ctypes and strings the per-protocol calls together
in the order DESIGN.md D3a-D3d fixes.  Pins: tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-Wall", "-o", _SO, _SRC])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        c = ctypes
        vp, u8p, i32p = c.c_void_p, c.c_char_p, c.c_void_p
        L.or_fr_op.argtypes = [c.c_int, vp, vp, vp]
        L.or_embed_i64.argtypes = [vp, c.c_uint64, vp]
        L.or_pinv.restype = c.c_uint64
        L.or_blake2s.argtypes = [vp, c.c_uint64, vp]
        L.or_transcript_init.argtypes = [vp, vp]
        L.or_transcript_absorb.argtypes = [vp, u8p, vp, c.c_uint64]
        L.or_transcript_challenges.argtypes = [vp, u8p, c.c_uint32, vp]
        L.or_beta.argtypes = [vp, vp, c.c_uint32, vp]
        L.or_eq_table.argtypes = [vp, c.c_uint32, vp]
        L.or_mle_fr.argtypes = [vp, c.c_uint32, vp, vp]
        L.or_mle_i32.argtypes = [i32p, c.c_uint32, vp, vp]
        L.or_sumcheck_prove.argtypes = [vp, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp, vp, vp]
        L.or_sumcheck_verify.argtypes = [vp, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp, vp]
        L.or_matmul_reduce.argtypes = [vp, i32p, i32p, c.c_uint32, c.c_uint32, c.c_uint32, c.c_uint32,
                                       c.c_int, c.c_int, vp, vp, vp, vp]
        L.or_relu_tables.argtypes = [i32p, i32p, c.c_uint64, c.c_uint32, c.c_uint32] + [vp] * 7
        L.or_relu_prove.argtypes = [vp, i32p, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp]
        L.or_loss_grad_prove.argtypes = [vp, c.c_uint32, i32p, i32p, i32p, vp, vp]
        L.or_relu_prove_pts.argtypes = [vp, i32p, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp, vp]
        L.or_claim_merge_prove.argtypes = [vp, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp, vp,
                                           vp, vp, vp, vp, vp, vp]
        L.or_relu_verify_pts.argtypes = [vp, i32p, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp]
        L.or_rescale_prove.argtypes = [vp, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.or_relu_verify.argtypes = [vp, i32p, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp]
        L.or_reindex_prove.argtypes = [vp, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp, vp, vp,
                                       vp, vp, vp, vp]
        L.or_relu_merge.argtypes = [vp, i32p, i32p, c.c_uint32, c.c_uint32, c.c_uint32, vp, vp, vp, vp, vp, vp, vp]
        L.or_zero_sumcheck_prove.argtypes = [vp, c.c_uint32, i32p, i32p, i32p, vp, vp, vp, vp]
        L.or_set_threads.argtypes = [c.c_int]
        L.or_get_threads.restype = c.c_int
        L.or_transcript_size.restype = c.c_uint64
        _lib = L
    return _lib


# ---------------------------------------------------------------- byte helpers
def to_bytes(vals) -> bytes:
    return b"".join((int(v) % P).to_bytes(32, "little") for v in vals)


def from_bytes(b: bytes, n: int | None = None) -> list:
    n = len(b) // 32 if n is None else n
    return [int.from_bytes(b[32 * i:32 * i + 32], "little") for i in range(n)]


def _buf(nbytes: int):
    return ctypes.create_string_buffer(max(1, nbytes))


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int):
    lib().or_set_threads(int(n))


def threads() -> int:
    return lib().or_get_threads()


# ---------------------------------------------------------------- field / hash
def fr_op(op: str, a: int, b: int | None = None) -> int:
    code = {"add": 0, "sub": 1, "mul": 2, "inv": 3, "neg": 4}[op]
    out = _buf(32)
    ab = a.to_bytes(32, "little") if a < (1 << 256) else None
    bb = None if b is None else b.to_bytes(32, "little")
    s = lib().or_fr_op(code, ab, bb, out)
    if s:
        raise ValueError(f"or_fr_op status {s}")
    return int.from_bytes(out.raw[:32], "little")


def embed(v) -> list:
    v = np.ascontiguousarray(np.asarray(v, dtype=np.int64).reshape(-1))
    out = _buf(32 * v.size)
    lib().or_embed_i64(_ptr(v), v.size, out)
    return from_bytes(out.raw[:32 * v.size])


def blake2s(msg: bytes) -> bytes:
    """BLAKE2s-256 (RFC 7693), the transcript hash H of DESIGN.md D3."""
    out = _buf(32)
    lib().or_blake2s(msg, len(msg), out)
    return out.raw[:32]


def pinv() -> int:
    return lib().or_pinv()


class Transcript:
    """Fiat-Shamir transcript (D3), state = 32 bytes."""

    def __init__(self, seed: bytes):
        assert len(seed) == 32
        self.st = _buf(32)
        lib().or_transcript_init(self.st, seed)

    def absorb(self, tag: str, msg: bytes):
        lib().or_transcript_absorb(self.st, tag.encode(), msg, len(msg))

    def challenges(self, tag: str, n: int) -> list:
        out = _buf(32 * n)
        lib().or_transcript_challenges(self.st, tag.encode(), n, out)
        return from_bytes(out.raw[:32 * n], n)

    def state(self) -> bytes:
        return self.st.raw[:32]


# ---------------------------------------------------------------- eq / MLE
def beta(u, v) -> int:
    out = _buf(32)
    s = lib().or_beta(to_bytes(u), to_bytes(v), len(u), out)
    if s:
        raise ValueError(s)
    return from_bytes(out.raw[:32])[0]


def eq_table(point) -> list:
    k = len(point)
    out = _buf(32 << k)
    lib().or_eq_table(to_bytes(point), k, out)
    return from_bytes(out.raw[:32 << k])


def mle_fr(table, point) -> int:
    m = len(point)
    assert len(table) == 1 << m
    out = _buf(32)
    lib().or_mle_fr(to_bytes(table), m, to_bytes(point), out)
    return from_bytes(out.raw[:32])[0]


def mle_i32(table: np.ndarray, point) -> int:
    t = np.ascontiguousarray(np.asarray(table, dtype=np.int32).reshape(-1))
    m = len(point)
    assert t.size == 1 << m
    out = _buf(32)
    lib().or_mle_i32(_ptr(t), m, to_bytes(point), out)
    return from_bytes(out.raw[:32])[0]


# ---------------------------------------------------------------- product sumcheck
def sumcheck_prove(tr: Transcript, m: int, n_eq: int, tables: list, w: list, claim: int | None = None):
    """Returns dict(claim, msgs[m][K+1], r[m], finals[K])."""
    K = len(tables)
    tb = b"".join(to_bytes(t) for t in tables)
    claim_out, msgs, r, fin = _buf(32), _buf(32 * m * (K + 1)), _buf(32 * m), _buf(32 * K)
    s = lib().or_sumcheck_prove(tr.st, m, n_eq, K, to_bytes(w), tb,
                                None if claim is None else to_bytes([claim]), claim_out, msgs, r, fin)
    if s:
        raise ValueError(f"or_sumcheck_prove status {s}")
    flat = from_bytes(msgs.raw[:32 * m * (K + 1)])
    return dict(claim=from_bytes(claim_out.raw[:32])[0],
                msgs=[flat[t * (K + 1):(t + 1) * (K + 1)] for t in range(m)],
                r=from_bytes(r.raw[:32 * m], m), finals=from_bytes(fin.raw[:32 * K], K))


def sumcheck_verify(tr: Transcript, m: int, n_eq: int, K: int, w: list, claim: int, msgs, finals,
                    tables: list | None = None):
    """0 = accept; >0 failing round (1-based); -100 final product; -200-k final of table k."""
    flat = [v for row in msgs for v in row]
    tb = None if tables is None else b"".join(to_bytes(t) for t in tables)
    r = _buf(32 * max(m, 1))
    s = lib().or_sumcheck_verify(tr.st, m, n_eq, K, to_bytes(w), to_bytes([claim]), to_bytes(flat),
                                 to_bytes(finals), tb, r)
    return s


# ---------------------------------------------------------------- matmul
def matmul_prove(tr: Transcript, A: np.ndarray, B: np.ndarray, transA=False, transB=False):
    """Oracle for zk_matmul_reduce + zk_sumcheck_prove (D3a).

    A: [N][D1][D2] int32 (or [N][D2][D1] if transA), B: [N][D2][D3] (or [N][D3][D2]).
    """
    A = np.ascontiguousarray(A, dtype=np.int32)
    B = np.ascontiguousarray(B, dtype=np.int32)
    N = A.shape[0]
    D1, D2 = (A.shape[2], A.shape[1]) if transA else (A.shape[1], A.shape[2])
    D3 = B.shape[1] if transB else B.shape[2]
    lg = [int(v).bit_length() - 1 for v in (N, D1, D2, D3)]
    for v, l in zip((N, D1, D2, D3), lg):
        assert v == 1 << l, "dimensions must be powers of two"
    logN, logD1, logD2, logD3 = lg
    npts = logN + logD1 + logD3
    pts, claim, At, Bt = _buf(32 * npts), _buf(32), _buf(32 * D2 * N), _buf(32 * D2 * N)
    s = lib().or_matmul_reduce(tr.st, _ptr(A), _ptr(B), logN, logD1, logD2, logD3, int(transA), int(transB),
                               pts, claim, At, Bt)
    if s:
        raise ValueError(f"or_matmul_reduce status {s}")
    P_ = from_bytes(pts.raw[:32 * npts], npts)
    w, u1, u3 = P_[:logN], P_[logN:logN + logD1], P_[logN + logD1:]
    claim_v = from_bytes(claim.raw[:32])[0]
    At_l = from_bytes(At.raw[:32 * D2 * N])
    Bt_l = from_bytes(Bt.raw[:32 * D2 * N])
    sc = sumcheck_prove(tr, logN + logD2, logN, [At_l, Bt_l], w, claim_v)
    return dict(logs=lg, w=w, u1=u1, u3=u3, claim=claim_v, At=At_l, Bt=Bt_l, **{k: sc[k] for k in ("msgs", "r", "finals")})


# ---------------------------------------------------------------- zkReLU
def relu_tables(Z: np.ndarray, GA: np.ndarray, Q: int, R: int):
    Z = np.ascontiguousarray(Z, dtype=np.int32).reshape(-1)
    GA = np.ascontiguousarray(GA, dtype=np.int32).reshape(-1)
    D = Z.size
    sign = np.zeros(D, np.uint8)
    outs = [np.zeros(D, np.int32) for _ in range(6)]
    s = lib().or_relu_tables(_ptr(Z), _ptr(GA), D, Q, R, _ptr(sign), *[_ptr(o) for o in outs])
    if s:
        raise ValueError(f"or_relu_tables status {s}")
    A, GZ, Zp, GAp, RZ, RGA = outs
    return dict(sign=sign, A=A, GZ=GZ, Zp=Zp, GAp=GAp, RZ=RZ, RGA=RGA)


def relu_logB(Q: int, R: int) -> int:
    return max(0, (Q + R - 1).bit_length())


def relu_prove(tr: Transcript, Z: np.ndarray, GA: np.ndarray, Q: int, R: int, points=None):
    """App. A zkReLU (D3b).  points: None (u_Z, u_A, u_GA, u_GZ drawn from the transcript) or the chained
    form (D25): the four logD-element points given (the window's merged claims)."""
    Z = np.ascontiguousarray(Z, dtype=np.int32).reshape(-1)
    GA = np.ascontiguousarray(GA, dtype=np.int32).reshape(-1)
    logD = Z.size.bit_length() - 1
    assert Z.size == 1 << logD
    logB = relu_logB(Q, R)
    m = logB + logD
    claims, chal, msgs, pt, fin = _buf(128), _buf(32 * (2 + m)), _buf(128 * m), _buf(32 * m), _buf(96)
    if points is None:
        s = lib().or_relu_prove(tr.st, _ptr(Z), _ptr(GA), logD, Q, R, claims, chal, msgs, pt, fin)
    else:
        assert len(points) == 4 and all(len(u) == logD for u in points)
        s = lib().or_relu_prove_pts(tr.st, _ptr(Z), _ptr(GA), logD, Q, R, to_bytes([x for u in points for x in u]),
                                    claims, chal, msgs, pt, fin)
    if s:
        raise ValueError(f"or_relu_prove status {s}")
    flat = from_bytes(msgs.raw[:128 * m])
    ch = from_bytes(chal.raw[:32 * (2 + m)])
    return dict(claims=from_bytes(claims.raw[:128]), r=ch[0], rp=ch[1], ubin=ch[2:],
                msgs=[flat[4 * t:4 * t + 4] for t in range(m)], point=from_bytes(pt.raw[:32 * m]),
                finals=from_bytes(fin.raw[:96]))


def relu_verify(tr: Transcript, Z, GA, Q: int, R: int, claims, msgs, finals, points=None) -> int:
    Zc = None if Z is None else np.ascontiguousarray(Z, dtype=np.int32).reshape(-1)
    Gc = None if GA is None else np.ascontiguousarray(GA, dtype=np.int32).reshape(-1)
    m = len(msgs)
    logD = m - relu_logB(Q, R)
    flat = [v for row in msgs for v in row]
    if points is not None:
        return lib().or_relu_verify_pts(tr.st, None if Zc is None else _ptr(Zc), None if Gc is None else _ptr(Gc),
                                        logD, Q, R, to_bytes([x for u in points for x in u]), to_bytes(claims),
                                        to_bytes(flat), to_bytes(finals))
    return lib().or_relu_verify(tr.st, None if Zc is None else _ptr(Zc), None if Gc is None else _ptr(Gc),
                                logD, Q, R, to_bytes(claims), to_bytes(flat), to_bytes(finals))


# ---------------------------------------------------------------- N1: re-indexing, aux-claim merge
def reindex_prove(tr: Transcript, X: np.ndarray, views: list, u: list, claims: list, want_tables: bool = False):
    """Eq. (sc-reindex) (D20).  X: [N][D] int32 (N, D powers of two); views: list of
    (map: int array of 2^{n_k} slice indices or -1 for an empty slot, u_k: n_k points); u: log2 D
    points; claims: c_k = X_k~(u, u_k).  Returns dict(rk, claim, msgs, r, finals[, C, Xu])."""
    X = np.ascontiguousarray(X, dtype=np.int32)
    N, D = X.shape
    n, d = N.bit_length() - 1, D.bit_length() - 1
    assert N == 1 << n and D == 1 << d
    K = len(views)
    nk = [len(m).bit_length() - 1 for m, _ in views]
    for (mp, uk), l in zip(views, nk):
        assert len(mp) == 1 << l and len(uk) == l
    maps = np.concatenate([np.asarray(mp, dtype=np.int64) & 0xFFFFFFFF for mp, _ in views]).astype(np.uint32)
    uk_all = [x for _, uk in views for x in uk]
    rk, claim, msgs, r, fin = _buf(32 * K), _buf(32), _buf(32 * 3 * max(n, 1)), _buf(32 * max(n, 1)), _buf(64)
    tabs = _buf(64 * N) if want_tables else None
    s = lib().or_reindex_prove(tr.st, _ptr(X), n, d, K, (ctypes.c_uint32 * K)(*nk), _ptr(maps), to_bytes(uk_all),
                               to_bytes(u), to_bytes(claims), rk, claim, msgs, r, fin, tabs)
    if s:
        raise ValueError(f"or_reindex_prove status {s}")
    flat = from_bytes(msgs.raw[:96 * n])
    out = dict(rk=from_bytes(rk.raw[:32 * K]), claim=from_bytes(claim.raw[:32])[0],
               msgs=[flat[3 * t:3 * t + 3] for t in range(n)], r=from_bytes(r.raw[:32 * n], n),
               finals=from_bytes(fin.raw[:64], 2))
    if want_tables:
        tv = from_bytes(tabs.raw[:64 * N])
        out["C"], out["Xu"] = tv[:N], tv[N:]
    return out


def relu_merge(tr: Transcript, Z: np.ndarray, GA: np.ndarray, Q: int, R: int, point: list, finals: list):
    """The zkReLU aux-claim merge (D21) after relu_prove on the same transcript.
    Returns dict(rho, claim, msgs, r, finals): finals[0] = aux~(r_s, v, r_j) (the merged claim)."""
    Z = np.ascontiguousarray(Z, dtype=np.int32).reshape(-1)
    GA = np.ascontiguousarray(GA, dtype=np.int32).reshape(-1)
    logD = Z.size.bit_length() - 1
    m = relu_logB(Q, R) + 1
    rho, claim, msgs, r, fin = _buf(32), _buf(32), _buf(96 * m), _buf(32 * m), _buf(64)
    s = lib().or_relu_merge(tr.st, _ptr(Z), _ptr(GA), logD, Q, R, to_bytes(point), to_bytes(finals), rho, claim,
                            msgs, r, fin)
    if s:
        raise ValueError(f"or_relu_merge status {s}")
    flat = from_bytes(msgs.raw[:96 * m])
    return dict(rho=from_bytes(rho.raw[:32])[0], claim=from_bytes(claim.raw[:32])[0],
                msgs=[flat[3 * t:3 * t + 3] for t in range(m)], r=from_bytes(r.raw[:32 * m], m),
                finals=from_bytes(fin.raw[:64], 2))


# ---------------------------------------------------------------- N2: Protocol 2 zero form
def zero_sumcheck_prove(tr: Transcript, Y: np.ndarray, A: np.ndarray, B: np.ndarray):
    """0 = sum_x beta(w, x) (Y(x) - A(x) B(x)) (Eq. tensor-op-aggr + Protocol 2, D22); int32
    tables of 2^m entries.  Returns dict(w, msgs[m][3], r, finals (Y~, A~, B~ at r))."""
    Y, A, B = (np.ascontiguousarray(t, dtype=np.int32).reshape(-1) for t in (Y, A, B))
    m = Y.size.bit_length() - 1
    assert Y.size == 1 << m and A.size == Y.size and B.size == Y.size
    w, msgs, r, fin = _buf(32 * m), _buf(96 * m), _buf(32 * m), _buf(96)
    s = lib().or_zero_sumcheck_prove(tr.st, m, _ptr(Y), _ptr(A), _ptr(B), w, msgs, r, fin)
    if s:
        raise ValueError(f"or_zero_sumcheck_prove status {s}")
    flat = from_bytes(msgs.raw[:96 * m])
    return dict(w=from_bytes(w.raw[:32 * m], m), msgs=[flat[3 * t:3 * t + 3] for t in range(m)],
                r=from_bytes(r.raw[:32 * m], m), finals=from_bytes(fin.raw[:96], 3))


# ---------------------------------------------------------------- N2: the loss-gradient family
def loss_grad_prove(tr: Transcript, GZ: np.ndarray, Z: np.ndarray, Y: np.ndarray):
    """Eq. (fcnn-GZ-last) G_Z = Z - Y (D24): returns dict(u, claims = [G_Z~(u), Z~(u), Y~(u)])."""
    GZ, Z, Y = (np.ascontiguousarray(t, dtype=np.int32).reshape(-1) for t in (GZ, Z, Y))
    m = Z.size.bit_length() - 1
    assert Z.size == 1 << m and GZ.size == Z.size and Y.size == Z.size
    u, cl = _buf(32 * m), _buf(96)
    s = lib().or_loss_grad_prove(tr.st, m, _ptr(GZ), _ptr(Z), _ptr(Y), u, cl)
    if s:
        raise ValueError(f"or_loss_grad_prove status {s}")
    return dict(u=from_bytes(u.raw[:32 * m], m), claims=from_bytes(cl.raw[:96], 3))


# ---------------------------------------------------------------- N3: the claim merge (D25)
def claim_merge_prove(tr: Transcript, X: np.ndarray, claims: list):
    """General Eq. (sc-reindex) (D25).  X: [N][D] int32 (powers of two).  claims: list of
    dicts(map = 2^{n_k} slice indices (-1: empty slot), u = n_k slot points, v = log2 D inner points,
    c = the claimed value X_k~(v, u)).  Returns dict(rho, A = dict(msgs, r, finals), B = dict(msgs, r,
    finals), point = r_B || r_A[:n], claim = finals_B[1]): the one claim X~(point) left on the stack."""
    X = np.ascontiguousarray(X, dtype=np.int32)
    N, D = X.shape
    n, d = N.bit_length() - 1, D.bit_length() - 1
    assert N == 1 << n and D == 1 << d
    K = len(claims)
    kap = max(0, (K - 1).bit_length())
    nk = [len(c["map"]).bit_length() - 1 for c in claims]
    for c, l in zip(claims, nk):
        assert len(c["map"]) == 1 << l and len(c["u"]) == l and len(c["v"]) == d
    maps = np.concatenate([np.asarray(c["map"], dtype=np.int64) & 0xFFFFFFFF for c in claims]).astype(np.uint32)
    mA = n + kap
    rho, mgA, rA, fA = _buf(32 * K), _buf(96 * mA), _buf(32 * mA), _buf(64)
    mgB, rB, fB = _buf(96 * d), _buf(32 * d), _buf(64)
    s = lib().or_claim_merge_prove(tr.st, _ptr(X), n, d, K, (ctypes.c_uint32 * K)(*nk), _ptr(maps),
                                   to_bytes([x for c in claims for x in c["u"]]),
                                   to_bytes([x for c in claims for x in c["v"]]), to_bytes([c["c"] for c in claims]),
                                   rho, mgA, rA, fA, mgB, rB, fB)
    if s:
        raise ValueError(f"or_claim_merge_prove status {s}")
    fa, fb = from_bytes(mgA.raw[:96 * mA]), from_bytes(mgB.raw[:96 * d])
    A = dict(msgs=[fa[3 * t:3 * t + 3] for t in range(mA)], r=from_bytes(rA.raw[:32 * mA], mA),
             finals=from_bytes(fA.raw[:64], 2))
    B = dict(msgs=[fb[3 * t:3 * t + 3] for t in range(d)], r=from_bytes(rB.raw[:32 * d], d),
             finals=from_bytes(fB.raw[:64], 2))
    return dict(rho=from_bytes(rho.raw[:32 * K], K), A=A, B=B, point=B["r"] + A["r"][:n], claim=B["finals"][1])


# ---------------------------------------------------------------- N2: the top-layer rescale (D26)
def rescale_prove(tr: Transcript, Z: np.ndarray, Q: int, R: int, points):
    """Z = 2^R Z' + R_Z through the bits of Z (D26) at the given points (u_Z, u_P).
    Returns dict(claims = [Z~(u_Z), Z'~(u_P)], r, A = dict(msgs, r, finals), w, B = dict(msgs, r, finals))."""
    Z = np.ascontiguousarray(Z, dtype=np.int32).reshape(-1)
    logD = Z.size.bit_length() - 1
    assert Z.size == 1 << logD and len(points) == 2 and all(len(u) == logD for u in points)
    m = relu_logB(Q, R) + logD
    cl, r, w = _buf(64), _buf(32), _buf(32 * m)
    mA, rA, fA, mB, rB, fB = _buf(96 * m), _buf(32 * m), _buf(64), _buf(96 * m), _buf(32 * m), _buf(64)
    s = lib().or_rescale_prove(tr.st, _ptr(Z), logD, Q, R, to_bytes(points[0] + points[1]), cl, r, mA, rA, fA, w,
                               mB, rB, fB)
    if s:
        raise ValueError(f"or_rescale_prove status {s}")
    fa, fb = from_bytes(mA.raw[:96 * m]), from_bytes(mB.raw[:96 * m])
    return dict(claims=from_bytes(cl.raw[:64], 2), r=from_bytes(r.raw[:32])[0], w=from_bytes(w.raw[:32 * m], m),
                A=dict(msgs=[fa[3 * t:3 * t + 3] for t in range(m)], r=from_bytes(rA.raw[:32 * m], m),
                       finals=from_bytes(fA.raw[:64], 2)),
                B=dict(msgs=[fb[3 * t:3 * t + 3] for t in range(m)], r=from_bytes(rB.raw[:32 * m], m),
                       finals=from_bytes(fB.raw[:64], 2)))
