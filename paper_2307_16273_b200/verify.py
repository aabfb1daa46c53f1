"""Host verifiers (D23): ctypes marshalling of libzkdl's zk_verify_* /
zk_htr_* (verify.cu, plain host code), and the window verifier that replays the D3d fork/join
transcripts of a FAC4DNN proving window.

Verification replays the prover's rounds; every round identity and each protocol's final
identity is checked here.  The finals are claims on the committed tensors (commitments: out of scope,
SURVEY §8(f) N4); `verify_window` returns them per family so a caller holding the tensors (tests) or
their commitments can close them.
"""
from __future__ import annotations

import ctypes

from ._lib import lib

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
ZK_OK, ZK_REJECT = 0, 1


def _fr(vals) -> ctypes.Array:
    b = b"".join(int(v).to_bytes(32, "little") for v in vals)
    return ctypes.create_string_buffer(b, max(1, len(b)))


def _ints(buf, n: int) -> list:
    raw = bytes(buf)[:32 * n]
    return [int.from_bytes(raw[32 * i:32 * i + 32], "little") for i in range(n)]


class HostTranscript:
    """The D3 transcript on a 32-byte host state (zk_htr_*)."""

    def __init__(self, seed: bytes | None = None, state: bytes | None = None):
        self.st = ctypes.create_string_buffer(32)
        if state is not None:
            assert len(state) == 32
            ctypes.memmove(self.st, state, 32)
        else:
            assert seed is not None and len(seed) == 32
            _check(lib().zk_htr_init(seed, self.st))

    def state(self) -> bytes:
        return self.st.raw

    def absorb(self, tag: str, msg: bytes) -> None:
        _check(lib().zk_htr_absorb(self.st, tag.encode(), msg, len(msg)))

    def challenges(self, tag: str, n: int) -> list:
        out = ctypes.create_string_buffer(32 * max(1, n))
        _check(lib().zk_htr_challenges(self.st, tag.encode(), n, out))
        return _ints(out, n)

    def fork(self, tag: str) -> "HostTranscript":
        """D3d: a child transcript seeded with the canonical bytes of this transcript's challenge."""
        return HostTranscript(seed=self.challenges(tag, 1)[0].to_bytes(32, "little"))


def _check(st: int) -> None:
    if st not in (ZK_OK, ZK_REJECT):
        raise ValueError(f"zk verifier error status {st}")


class Rejected(Exception):
    def __init__(self, what: str, where: int):
        super().__init__(f"{what}: rejected at {where} (round, or -100 final identity, -1 claim, -101 weights)")
        self.where = where


def _run(what: str, fn, *args) -> None:
    fail = ctypes.c_int32(0)
    st = fn(*args, ctypes.byref(fail))
    _check(st)
    if st == ZK_REJECT:
        raise Rejected(what, fail.value)


def verify_sumcheck(tr: HostTranscript, proof: bytes, w: list, claim: int | None = None) -> list:
    """zk_verify_sumcheck: returns the point r; raises Rejected."""
    m = int.from_bytes(proof[:4], "little")
    pt = ctypes.create_string_buffer(32 * m)
    _run("sumcheck", lib().zk_verify_sumcheck, tr.st, proof, len(proof), _fr(w),
         None if claim is None else _fr([claim]), pt)
    return _ints(pt, m)


def verify_hadamard_zero(tr: HostTranscript, proof: bytes) -> dict:
    m = int.from_bytes(proof[:4], "little")
    w, pt = ctypes.create_string_buffer(32 * m), ctypes.create_string_buffer(32 * m)
    _run("hadamard zero", lib().zk_verify_hadamard_zero, tr.st, proof, len(proof), w, pt)
    return dict(w=_ints(w, m), r=_ints(pt, m))


def verify_relu(tr: HostTranscript, proof: bytes) -> list:
    logD, Q, R = (int.from_bytes(proof[4 * i:4 * i + 4], "little") for i in range(3))
    m = max(0, (Q + R - 1).bit_length()) + logD
    pt = ctypes.create_string_buffer(32 * m)
    _run("zkReLU", lib().zk_verify_relu, tr.st, proof, len(proof), pt)
    return _ints(pt, m)


def verify_loss_grad(tr: HostTranscript, m: int, claims: list) -> list:
    """zk_verify_loss_grad (D24): returns the point u; raises Rejected unless G_Z~(u) = Z~(u) - Y~(u)."""
    pt = ctypes.create_string_buffer(32 * m)
    _run("loss gradient", lib().zk_verify_loss_grad, tr.st, m, _fr(claims), pt)
    return _ints(pt, m)


def verify_relu_merge(tr: HostTranscript, logD: int, Q: int, R: int, relu_point: list, relu_finals: list,
                      proof: bytes) -> list:
    m = max(0, (Q + R - 1).bit_length()) + 1
    pt = ctypes.create_string_buffer(32 * m)
    _run("zkReLU merge", lib().zk_verify_relu_merge, tr.st, logD, Q, R, _fr(relu_point), _fr(relu_finals), proof,
         len(proof), pt)
    return _ints(pt, m)


def verify_matmul(tr: HostTranscript, logs, res: dict) -> list:
    """A matmul family (rows a3-a6): the verifier draws w, u1, u3 itself (D3a), checks they are the
    prover's, then verifies the product sumcheck (n_eq = logN) of the claim Y~(w, u1, u3)."""
    lN, l1, l2, l3 = logs
    tr.absorb("mm/hdr", b"".join(int(v).to_bytes(4, "little") for v in (lN, l1, l2, l3)))
    w, u1, u3 = tr.challenges("mm/w", lN), tr.challenges("mm/u1", l1), tr.challenges("mm/u3", l3)
    if (w, u1, u3) != (res["w"], res["u1"], res["u3"]):
        raise Rejected("matmul points", -2)
    return verify_sumcheck(tr, res["proof"], w, res["claim"])


def verify_window(seed: bytes, header: bytes, families: list, results: list) -> list:
    """Replays a window (D3d): W absorbs "fcn/hdr", per family "fcn/fam" and forks "fcn/fork"; each
    family's proof is verified on its own forked transcript and must end in the state the prover
    reported; W absorbs "fcn/join" of every family and must end in the reported window state.
    families: the window's family records (shapes only are read); results: fcn.prove_window's output.
    Returns per family the claims left for the commitments: {name, point, finals}."""
    from .api import _mm_logs
    W = HostTranscript(seed=seed)
    W.absorb("fcn/hdr", header)
    kids = []
    for f in families:
        W.absorb("fcn/fam", f.name.encode())
        kids.append(W.fork("fcn/fork"))
    out = []
    for f, T, res in zip(families, kids, results):
        if hasattr(f, "A"):   # a matmul family (device record or host synth.fcn record: shapes only)
            ta, tb = getattr(f, "trans_a", getattr(f, "transA", False)), getattr(f, "trans_b", getattr(f, "transB", False))
            r = verify_matmul(T, _mm_logs(f.A, f.B, ta, tb), res)
            out.append(dict(name=f.name, point=r, finals=res["finals"]))
        else:
            logD = int.from_bytes(res["proof"][:4], "little")
            r = verify_relu(T, res["proof"])
            item = dict(name=f.name, point=r, finals=res["finals"])
            if "merge" in res:
                item["merge_point"] = verify_relu_merge(T, logD, f.Q, f.R, r, res["finals"], res["merge"]["proof"])
                item["merge_finals"] = res["merge"]["finals"]
            out.append(item)
        if T.state() != res["state"]:
            raise Rejected(f"family {f.name} transcript state", -3)
    for T in kids:
        W.absorb("fcn/join", T.state())
    if W.state() != results[-1]["window_state"]:
        raise Rejected("window transcript state", -3)
    return out
