"""Thin Python binding of libzkdl (include/zkdl.h) — argument marshalling only.

Every step of the proving path runs in the library's CUDA kernels; torch is
used for device memory and streams.  Field elements are Python ints in
[0, p); device Fr tables are torch.uint8 tensors of shape [n, 32] holding the
library's internal (Montgomery) representation.  Function names follow the
ABI with the ``zk_`` prefix dropped.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import CmView, MmShape, ProdStmt, View, ZkError, lib

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def _fr_buf(vals) -> ctypes.Array:
    b = b"".join((int(v) % P).to_bytes(32, "little") for v in vals)
    return ctypes.create_string_buffer(b, max(1, len(b)))


def _ints(buf, n: int) -> list:
    raw = bytes(buf)[:32 * n]
    return [int.from_bytes(raw[32 * i:32 * i + 32], "little") for i in range(n)]


def _dev_ptr(t: torch.Tensor, dtype=None) -> int:
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"expected {dtype}, got {t.dtype}")
    return t.data_ptr()


class Context:
    """zk_ctx: a device, a CUDA stream (torch's current stream by default), the last error."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = ctypes.c_void_p()
        st = lib().zk_ctx_create(device, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if st != 0:
            raise ZkError(st, "zk_ctx_create failed (no sm_100 CUDA device?)")
        self.h = h

    def check(self, st: int):
        if st != 0:
            raise ZkError(st, lib().zk_last_error(self.h).decode())

    @property
    def launches(self) -> int:
        return int(lib().zk_ctx_launch_count(self.h))

    def synchronize(self):
        self.check(lib().zk_ctx_synchronize(self.h))

    def set_persistent(self, allow: bool):
        """zk_ctx_set_persistent: allow / forbid this context's persistent (spin-waiting) sumcheck kernels."""
        self.check(lib().zk_ctx_set_persistent(self.h, 1 if allow else 0))

    def set_sm_budget(self, sms: int):
        """zk_ctx_set_sm_budget: cap the grid of this context's persistent kernels (0 = every SM)."""
        self.check(lib().zk_ctx_set_sm_budget(self.h, int(sms)))

    def profile(self, enable: bool):
        self.check(lib().zk_ctx_profile(self.h, int(enable)))

    def profile_filter(self, prefix: str | None):
        self.check(lib().zk_ctx_profile_filter(self.h, prefix.encode() if prefix else None))

    def profile_read(self) -> dict:
        """{kernel name: (launches, total_ms)} since the last read (synchronises)."""
        buf = ctypes.create_string_buffer(1 << 16)
        self.check(lib().zk_ctx_profile_read(self.h, buf, len(buf)))
        out = {}
        for line in buf.value.decode().splitlines():
            name, n, ms = line.split("\t")
            out[name] = (int(n), float(ms))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().zk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Transcript:
    """zk_transcript: device-resident Fiat-Shamir state (D3)."""

    def __init__(self, ctx: Context, seed: bytes | None, _handle=None):
        self.ctx = ctx
        if _handle is not None:
            self.h = _handle
            return
        assert len(seed) == 32
        h = ctypes.c_void_p()
        ctx.check(lib().zk_transcript_new(ctx.h, seed, ctypes.byref(h)))
        self.h = h

    def fork(self, tag: str, ctx: Context | None = None) -> "Transcript":
        """D3d fork: a child transcript seeded with this transcript's challenge `tag`, bound to `ctx`
        (its stream; default this transcript's).  Enqueued on this transcript's stream."""
        h = ctypes.c_void_p()
        child_ctx = ctx if ctx is not None else self.ctx
        self.ctx.check(lib().zk_transcript_fork(self.h, tag.encode(), child_ctx.h, ctypes.byref(h)))
        return Transcript(child_ctx, None, _handle=h)

    def absorb_state(self, tag: str, other: "Transcript"):
        """absorb(tag, other's 32-byte state), device to device (D3d join)."""
        self.ctx.check(lib().zk_transcript_absorb_state(self.h, tag.encode(), other.h))

    def absorb(self, tag: str, msg: bytes):
        self.ctx.check(lib().zk_transcript_absorb(self.h, tag.encode(), msg, len(msg)))

    def challenges(self, tag: str, n: int) -> list:
        out = ctypes.create_string_buffer(max(1, 32 * n))
        self.ctx.check(lib().zk_transcript_challenges(self.h, tag.encode(), n, out))
        return _ints(out, n)

    def state(self) -> bytes:
        out = ctypes.create_string_buffer(32)
        self.ctx.check(lib().zk_transcript_state(self.h, out))
        return out.raw[:32]

    def state_dev(self, out: torch.Tensor):
        """Stream-ordered copy of the state into 32 bytes of device memory (no synchronisation)."""
        assert out.dtype == torch.uint8 and out.numel() >= 32 and out.is_contiguous()
        self.ctx.check(lib().zk_transcript_state_dev(self.h, out.data_ptr()))

    def close(self):
        if getattr(self, "h", None):
            lib().zk_transcript_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- tables (rows a1, a2)
def fr_empty(n: int, device) -> torch.Tensor:
    return torch.empty((n, 32), dtype=torch.uint8, device=device)


def embed_i32(ctx: Context, t: torch.Tensor) -> torch.Tensor:
    out = fr_empty(t.numel(), t.device)
    ctx.check(lib().zk_embed_i32(ctx.h, _dev_ptr(t, torch.int32), t.numel(), out.data_ptr()))
    return out


def eq_table(ctx: Context, point: list, scale: int | None = None, device="cuda") -> torch.Tensor:
    k = len(point)
    out = fr_empty(1 << k, device)
    sc = _fr_buf([scale]) if scale is not None else None
    ctx.check(lib().zk_eq_table(ctx.h, _fr_buf(point), k, sc, out.data_ptr()))
    return out


def mle_eval_i32(ctx: Context, tab: torch.Tensor, point: list) -> int:
    out = ctypes.create_string_buffer(32)
    ctx.check(lib().zk_mle_eval_i32(ctx.h, _dev_ptr(tab, torch.int32), len(point), _fr_buf(point), out))
    return _ints(out, 1)[0]


def mle_eval_fr(ctx: Context, tab: torch.Tensor, point: list) -> int:
    out = ctypes.create_string_buffer(32)
    ctx.check(lib().zk_mle_eval_fr(ctx.h, _dev_ptr(tab, torch.uint8), len(point), _fr_buf(point), out))
    return _ints(out, 1)[0]


def fr_table_to_canonical(ctx: Context, tab: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(tab)
    ctx.check(lib().zk_fr_table_to_canonical(ctx.h, _dev_ptr(tab, torch.uint8), tab.shape[0], out.data_ptr()))
    return out


def fr_table_from_canonical(ctx: Context, tab: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(tab)
    ctx.check(lib().zk_fr_table_from_canonical(ctx.h, _dev_ptr(tab, torch.uint8), tab.shape[0], out.data_ptr()))
    return out


def fr_table_to_ints(ctx: Context, tab: torch.Tensor) -> list:
    raw = fr_table_to_canonical(ctx, tab).cpu().numpy().tobytes()
    return [int.from_bytes(raw[32 * i:32 * i + 32], "little") for i in range(tab.shape[0])]


def fr_table_from_ints(ctx: Context, vals, device="cuda") -> torch.Tensor:
    raw = b"".join((int(v) % P).to_bytes(32, "little") for v in vals)
    t = torch.frombuffer(bytearray(raw), dtype=torch.uint8).reshape(-1, 32).to(device)
    return fr_table_from_canonical(ctx, t)


# ---------------------------------------------------------------- matmul (row a3)
def _log2(n: int) -> int:
    l = n.bit_length() - 1
    if n != 1 << l:
        raise ValueError(f"{n} is not a power of two")
    return l


def matmul_reduce(ctx: Context, tr: Transcript, A: torch.Tensor, B: torch.Tensor, trans_a=False, trans_b=False):
    """A: [N][D1][D2] (or [N][D2][D1]), B: [N][D2][D3] (or [N][D3][D2]) int32 on the device."""
    N = A.shape[0]
    D1, D2 = (A.shape[2], A.shape[1]) if trans_a else (A.shape[1], A.shape[2])
    D3 = B.shape[1] if trans_b else B.shape[2]
    lN, l1, l2, l3 = (_log2(int(v)) for v in (N, D1, D2, D3))
    At = fr_empty(D2 * N, A.device)
    Bt = fr_empty(D2 * N, A.device)
    np_ = lN + l1 + l3
    pts = ctypes.create_string_buffer(max(32, 32 * np_))
    claim = ctypes.create_string_buffer(32)
    sh = MmShape(lN, l1, l2, l3, int(trans_a), int(trans_b))
    ctx.check(lib().zk_matmul_reduce(ctx.h, tr.h, _dev_ptr(A, torch.int32), _dev_ptr(B, torch.int32), sh,
                                     At.data_ptr(), Bt.data_ptr(), pts, claim))
    P_ = _ints(pts, np_)
    return dict(logs=(lN, l1, l2, l3), At=At, Bt=Bt, w=P_[:lN], u1=P_[lN:lN + l1], u3=P_[lN + l1:],
                claim=_ints(claim, 1)[0])


# ---------------------------------------------------------------- product sumcheck (rows a4-a6)
def parse_sumcheck_proof(raw: bytes) -> dict:
    m, n_eq, K = (int.from_bytes(raw[4 * i:4 * i + 4], "little") for i in range(3))
    vals = [int.from_bytes(raw[12 + 32 * i:44 + 32 * i], "little") for i in range((len(raw) - 12) // 32)]
    claim = vals[0]
    msgs = [vals[1 + t * (K + 1):1 + (t + 1) * (K + 1)] for t in range(m)]
    finals = vals[1 + m * (K + 1):1 + m * (K + 1) + K]
    return dict(m=m, n_eq=n_eq, K=K, claim=claim, msgs=msgs, finals=finals)


def sumcheck_prove(ctx: Context, tr: Transcript, m: int, n_eq: int, tables: list, w: list, claim: int | None = None):
    """tables: Fr tables ([2^m, 32] uint8, Montgomery) or int32 tables of 2^m entries."""
    K = len(tables)
    mask = 0
    ptrs = (ctypes.c_void_p * K)()
    for k, t in enumerate(tables):
        if t.dtype == torch.int32:
            mask |= 1 << k
            assert t.numel() == 1 << m
        else:
            assert t.dtype == torch.uint8 and t.shape == (1 << m, 32)
        ptrs[k] = _dev_ptr(t)
    wbuf = _fr_buf(w)
    stmt = ProdStmt(m, n_eq, K, mask, ctypes.cast(wbuf, ctypes.c_void_p))
    plen = ctypes.c_uint64(12 + 32 + 32 * m * (K + 1) + 32 * K)
    proof = ctypes.create_string_buffer(plen.value)
    point = ctypes.create_string_buffer(32 * m)
    cbuf = _fr_buf([claim]) if claim is not None else None
    ctx.check(lib().zk_sumcheck_prove(ctx.h, tr.h, ctypes.byref(stmt), ptrs, cbuf, None, proof, ctypes.byref(plen),
                                      point, None))
    res = parse_sumcheck_proof(proof.raw[:plen.value])
    res["r"] = _ints(point, m)
    res["proof"] = proof.raw[:plen.value]
    return res


# ---------------------------------------------------------------- zkReLU (rows a7, a8)
def relu_tables(ctx: Context, Z: torch.Tensor, GA: torch.Tensor, Q: int = 16, R: int = 16, extras: bool = True):
    D = Z.numel()
    dev = Z.device
    sign = torch.empty(D, dtype=torch.uint8, device=dev)
    outs = {k: torch.empty(D, dtype=torch.int32, device=dev) for k in ("A", "GZ", "Zp", "GAp", "RZ", "RGA")}
    ex = [outs[k].data_ptr() if extras else None for k in ("Zp", "GAp", "RZ", "RGA")]
    ctx.check(lib().zk_relu_tables(ctx.h, _dev_ptr(Z, torch.int32), _dev_ptr(GA, torch.int32), D, Q, R,
                                   sign.data_ptr(), outs["A"].data_ptr(), outs["GZ"].data_ptr(), *ex))
    outs["sign"] = sign
    return outs


def relu_logB(Q: int, R: int) -> int:
    return max(0, (Q + R - 1).bit_length())


def parse_relu_proof(raw: bytes, logB: int) -> dict:
    logD, Q, R = (int.from_bytes(raw[4 * i:4 * i + 4], "little") for i in range(3))
    vals = [int.from_bytes(raw[12 + 32 * i:44 + 32 * i], "little") for i in range((len(raw) - 12) // 32)]
    m = logB + logD
    return dict(logD=logD, Q=Q, R=R, claims=vals[:4], msgs=[vals[4 + 4 * t:8 + 4 * t] for t in range(m)],
                finals=vals[4 + 4 * m:7 + 4 * m])


def relu_prove(ctx: Context, tr: Transcript, Z: torch.Tensor, GA: torch.Tensor, Q: int = 16, R: int = 16):
    D = Z.numel()
    logD = _log2(D)
    logB = relu_logB(Q, R)
    plen = ctypes.c_uint64(12 + 128 + 128 * (logB + logD) + 96)
    proof = ctypes.create_string_buffer(plen.value)
    point = ctypes.create_string_buffer(32 * (logB + logD))
    ctx.check(lib().zk_relu_prove(ctx.h, tr.h, _dev_ptr(Z, torch.int32), _dev_ptr(GA, torch.int32), logD, Q, R, proof,
                                  ctypes.byref(plen), None, point, None))
    res = parse_relu_proof(proof.raw[:plen.value], logB)
    res["point"] = _ints(point, logB + logD)
    res["proof"] = proof.raw[:plen.value]
    return res


# ---------------------------------------------------------------- device-output provers (asynchronous)
def _a16(n: int) -> int:
    return (n + 15) & ~15


def _mm_logs(A: torch.Tensor, B: torch.Tensor, trans_a: bool, trans_b: bool):
    N = A.shape[0]
    D1, D2 = (A.shape[2], A.shape[1]) if trans_a else (A.shape[1], A.shape[2])
    D3 = B.shape[1] if trans_b else B.shape[2]
    return tuple(_log2(int(v)) for v in (N, D1, D2, D3))


def matmul_prove_len(logs) -> int:
    lN, l1, l2, l3 = logs
    m = lN + l2
    return _a16(32 * (lN + l1 + l3) + 32 + (12 + 32 + 32 * m * 3 + 64)) + 32 * m


def matmul_prove(ctx: Context, tr: Transcript, A: torch.Tensor, B: torch.Tensor, trans_a=False, trans_b=False,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_matmul_prove: reduce + product sumcheck, every output in device memory (no host sync).
    Returns the uint8 device buffer (layout in include/zkdl.h; parse with parse_matmul_out)."""
    logs = _mm_logs(A, B, trans_a, trans_b)
    n = matmul_prove_len(logs)
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=A.device)
    assert out.dtype == torch.uint8 and out.numel() >= n and out.is_contiguous()
    ln = ctypes.c_uint64(out.numel())
    sh = MmShape(*logs, int(trans_a), int(trans_b))
    ctx.check(lib().zk_matmul_prove(ctx.h, tr.h, _dev_ptr(A, torch.int32), _dev_ptr(B, torch.int32), sh, None, None,
                                    out.data_ptr(), ctypes.byref(ln)))
    return out


def parse_matmul_out(raw: bytes, logs) -> dict:
    lN, l1, l2, l3 = logs
    np_, m = lN + l1 + l3, lN + l2
    pts = [int.from_bytes(raw[32 * i:32 * i + 32], "little") for i in range(np_ + 1)]
    off = 32 * np_ + 32
    plen = 12 + 32 + 32 * m * 3 + 64
    res = parse_sumcheck_proof(raw[off:off + plen])
    res["proof"] = raw[off:off + plen]
    o_r = _a16(off + plen)
    res["r"] = [int.from_bytes(raw[o_r + 32 * i:o_r + 32 * i + 32], "little") for i in range(m)]
    res.update(w=pts[:lN], u1=pts[lN:lN + l1], u3=pts[lN + l1:np_], claim=pts[np_])
    return res


def relu_prove_len(logD: int, Q: int, R: int) -> int:
    logB = relu_logB(Q, R)
    return _a16(12 + 128 + 128 * (logB + logD) + 96) + 32 * (logB + logD)


def relu_prove_dev(ctx: Context, tr: Transcript, Z: torch.Tensor, GA: torch.Tensor, Q: int, R: int,
                   range_flag: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_relu_prove_dev: the zkReLU proof and point into a device buffer (no host sync); bit 0 of
    range_flag (int32 device scalar) is set when an input is out of range."""
    logD = _log2(Z.numel())
    n = relu_prove_len(logD, Q, R)
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=Z.device)
    assert out.dtype == torch.uint8 and out.numel() >= n and out.is_contiguous()
    assert range_flag.dtype == torch.int32 and range_flag.is_cuda
    ln = ctypes.c_uint64(out.numel())
    ctx.check(lib().zk_relu_prove_dev(ctx.h, tr.h, _dev_ptr(Z, torch.int32), _dev_ptr(GA, torch.int32), logD, Q, R,
                                      out.data_ptr(), ctypes.byref(ln), range_flag.data_ptr()))
    return out


def parse_relu_out(raw: bytes, logD: int, Q: int, R: int) -> dict:
    logB = relu_logB(Q, R)
    plen = 12 + 128 + 128 * (logB + logD) + 96
    res = parse_relu_proof(raw[:plen], logB)
    res["proof"] = raw[:plen]
    o_p = _a16(plen)
    res["point"] = [int.from_bytes(raw[o_p + 32 * i:o_p + 32 * i + 32], "little") for i in range(logB + logD)]
    return res


# ---------------------------------------------------------------- diagnostics
def diag_fr_op(ctx: Context, op: str, a: torch.Tensor, b: torch.Tensor | None = None) -> torch.Tensor:
    code = {"add": 0, "sub": 1, "mul": 2, "inv": 3, "neg": 4, "sqr": 5, "inv_bgcd": 6}[op]
    out = torch.empty_like(a)
    ctx.check(lib().zk_diag_fr_op(ctx.h, code, _dev_ptr(a), None if b is None else _dev_ptr(b), a.shape[0],
                                  out.data_ptr()))
    return out


def diag_mul_bench(ctx: Context, seed: torch.Tensor, iters: int, blocks: int) -> torch.Tensor:
    out = fr_empty(blocks * 256, seed.device)
    ctx.check(lib().zk_diag_mul_bench(ctx.h, _dev_ptr(seed), iters, blocks, out.data_ptr()))
    return out


# ---------------------------------------------------------------- SURVEY §8(f) N1
def reindex_prove(ctx: Context, tr: Transcript, X: torch.Tensor, views: list, u: list, claims: list) -> dict:
    """zk_reindex_prove (Eq. sc-reindex, D20).  X: int32 device tensor [N][D]; views: list of
    (map: sequence of 2^n_k slice indices, -1 = empty slot, u_k: n_k field elements); u: log2 D
    elements; claims: X_k~(u, u_k).  Returns dict(claim, msgs, r, finals, proof)."""
    assert X.dtype == torch.int32 and X.dim() == 2 and X.is_cuda
    N, D = X.shape
    n, d = _log2(N), _log2(D)
    K = len(views)
    keep = []
    vs = (View * K)()
    for k, (mp, uk) in enumerate(views):
        arr = (ctypes.c_uint32 * len(mp))(*[(int(i) & 0xFFFFFFFF) for i in mp])
        ub = _fr_buf(uk) if len(uk) else None
        keep += [arr, ub]
        vs[k] = View(_log2(len(mp)), ctypes.cast(arr, ctypes.c_void_p), ctypes.cast(ub, ctypes.c_void_p) if ub else None)
    plen = ctypes.c_uint64(12 + 32 + 32 * n * 3 + 64)
    proof = ctypes.create_string_buffer(plen.value)
    point = ctypes.create_string_buffer(32 * n)
    fin = ctypes.create_string_buffer(64)
    ctx.check(lib().zk_reindex_prove(ctx.h, tr.h, _dev_ptr(X, torch.int32), n, d, K, vs, _fr_buf(u) if d else None,
                                     _fr_buf(claims), proof, ctypes.byref(plen), point, fin))
    res = parse_sumcheck_proof(proof.raw[:plen.value])
    res["r"] = _ints(point, n)
    res["proof"] = proof.raw[:plen.value]
    return res


def relu_merge(ctx: Context, tr: Transcript, Z: torch.Tensor, GA: torch.Tensor, Q: int, R: int, point: list,
               finals: list) -> dict:
    """zk_relu_merge (D21) after relu_prove on the same transcript.  Returns
    dict(claim, msgs, r, finals, proof): finals[0] = aux~(r_s, v, r_j), the merged claim."""
    logD = _log2(Z.numel())
    m = relu_logB(Q, R) + 1
    plen = ctypes.c_uint64(12 + 32 + 32 * m * 3 + 64)
    proof = ctypes.create_string_buffer(plen.value)
    pt = ctypes.create_string_buffer(32 * m)
    fin = ctypes.create_string_buffer(64)
    ctx.check(lib().zk_relu_merge(ctx.h, tr.h, _dev_ptr(Z, torch.int32), _dev_ptr(GA, torch.int32), logD, Q, R,
                                  _fr_buf(point), _fr_buf(finals), proof, ctypes.byref(plen), pt, fin))
    res = parse_sumcheck_proof(proof.raw[:plen.value])
    res["r"] = _ints(pt, m)
    res["proof"] = proof.raw[:plen.value]
    return res


def relu_merge_len(Q: int, R: int) -> int:
    m = relu_logB(Q, R) + 1
    return _a16(12 + 32 + 96 * m + 64) + 32 * m


def relu_merge_dev(ctx: Context, tr: Transcript, Z: torch.Tensor, GA: torch.Tensor, Q: int, R: int,
                   relu_out: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_relu_merge_dev: the aux-claim merge from a zk_relu_prove_dev output, into a device buffer."""
    logD = _log2(Z.numel())
    n = relu_merge_len(Q, R)
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=Z.device)
    assert out.dtype == torch.uint8 and out.numel() >= n and out.is_contiguous()
    ln = ctypes.c_uint64(out.numel())
    ctx.check(lib().zk_relu_merge_dev(ctx.h, tr.h, _dev_ptr(Z, torch.int32), _dev_ptr(GA, torch.int32), logD, Q, R,
                                      relu_out.data_ptr(), out.data_ptr(), ctypes.byref(ln)))
    return out


def parse_relu_merge_out(raw: bytes, Q: int, R: int) -> dict:
    m = relu_logB(Q, R) + 1
    plen = 12 + 32 + 96 * m + 64
    res = parse_sumcheck_proof(raw[:plen])
    res["proof"] = raw[:plen]
    o = _a16(plen)
    res["r"] = [int.from_bytes(raw[o + 32 * i:o + 32 * i + 32], "little") for i in range(m)]
    return res


# ---------------------------------------------------------------- SURVEY §8(f) N2
def hadamard_zero_prove(ctx: Context, tr: Transcript, Y: torch.Tensor, A: torch.Tensor, B: torch.Tensor) -> dict:
    """zk_hadamard_zero_prove (Protocol 2's zero form, D22): int32 device tables of 2^m entries.
    Returns dict(w, msgs[m][3], r, finals (Y~, A~, B~ at r), proof)."""
    m = _log2(Y.numel())
    assert A.numel() == Y.numel() and B.numel() == Y.numel()
    plen = ctypes.c_uint64(4 + 96 * m + 96)
    proof = ctypes.create_string_buffer(plen.value)
    w, pt, fin = ctypes.create_string_buffer(32 * m), ctypes.create_string_buffer(32 * m), ctypes.create_string_buffer(96)
    ctx.check(lib().zk_hadamard_zero_prove(ctx.h, tr.h, _dev_ptr(Y, torch.int32), _dev_ptr(A, torch.int32),
                                           _dev_ptr(B, torch.int32), m, proof, ctypes.byref(plen), w, pt, fin))
    raw = proof.raw[:plen.value]
    vals = [int.from_bytes(raw[4 + 32 * i:36 + 32 * i], "little") for i in range(3 * m + 3)]
    return dict(w=_ints(w, m), msgs=[vals[3 * t:3 * t + 3] for t in range(m)], r=_ints(pt, m), finals=vals[3 * m:],
                proof=raw)


def loss_grad_prove(ctx: Context, tr: Transcript, GZ: torch.Tensor, Z: torch.Tensor, Y: torch.Tensor) -> dict:
    """zk_loss_grad_prove (Eq. fcnn-GZ-last, D24): int32 device tables of 2^m entries.
    Returns dict(u, claims = [G_Z~(u), Z~(u), Y~(u)])."""
    m = _log2(Z.numel())
    assert GZ.numel() == Z.numel() and Y.numel() == Z.numel()
    pt, cl = ctypes.create_string_buffer(32 * m), ctypes.create_string_buffer(96)
    ctx.check(lib().zk_loss_grad_prove(ctx.h, tr.h, _dev_ptr(GZ, torch.int32), _dev_ptr(Z, torch.int32),
                                       _dev_ptr(Y, torch.int32), m, pt, cl))
    return dict(u=_ints(pt, m), claims=_ints(cl, 3))


# ---------------------------------------------------------------- N3: the claim merge (D25)
CM_SOURCE = {"plain": 0, "relu_A": 1, "relu_GZ": 2, "bits": 3}


def claim_merge_layout(n: int, K: int, d: int) -> dict:
    """Byte offsets of a zk_claim_merge_dev output (include/zkdl.h)."""
    kap = max(0, (K - 1).bit_length())
    la, lb = 12 + 32 + 96 * (n + kap) + 64, 12 + 32 + 96 * d + 64
    off_pa = _a16(la + lb)
    off_pb = off_pa + 32 * (n + kap)
    off_pt = off_pb + 32 * d
    off_c = off_pt + 32 * (d + n)
    return dict(kappa=kap, la=la, lb=lb, off_pa=off_pa, off_pb=off_pb, off_pt=off_pt, off_c=off_c, total=off_c + 32)


def claim_merge_dev(ctx: Context, tr: Transcript, X: torch.Tensor, n: int, log_rows: int, log_cols: int, maps: list,
                    d_pts: torch.Tensor, d_claims: torch.Tensor, source: str = "plain", X2: torch.Tensor | None = None,
                    R: int = 0, out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_claim_merge_dev: maps = one slot->slice list per claim (-1: empty slot); d_pts / d_claims: device
    canonical bytes (per claim its inner point then its slot point; the claimed values).  Asynchronous;
    returns the uint8 output buffer (layout: claim_merge_layout)."""
    K = len(maps)
    lay = claim_merge_layout(n, K, log_rows + log_cols)
    if out is None:
        out = torch.empty(lay["total"], dtype=torch.uint8, device=X.device)
    assert out.dtype == torch.uint8 and out.numel() >= lay["total"] and out.is_contiguous()
    arrs = [(ctypes.c_uint32 * len(m))(*[int(i) & 0xFFFFFFFF for i in m]) for m in maps]
    views = (CmView * K)(*[CmView(len(m).bit_length() - 1, ctypes.cast(a, ctypes.c_void_p)) for m, a in zip(maps, arrs)])
    ln = ctypes.c_uint64(out.numel())
    ctx.check(lib().zk_claim_merge_dev(ctx.h, tr.h, _dev_ptr(X, torch.int32), None if X2 is None else _dev_ptr(X2, torch.int32),
                                       CM_SOURCE[source], R, n, log_rows, log_cols, K, views, _dev_ptr(d_pts, torch.uint8),
                                       _dev_ptr(d_claims, torch.uint8), out.data_ptr(), ctypes.byref(ln)))
    return out


def parse_claim_merge_out(raw: bytes, n: int, K: int, d: int) -> dict:
    lay = claim_merge_layout(n, K, d)
    A = parse_sumcheck_proof(raw[:lay["la"]])
    B = parse_sumcheck_proof(raw[lay["la"]:lay["la"] + lay["lb"]])
    mA = n + lay["kappa"]

    def pts(o, k):
        return [int.from_bytes(raw[o + 32 * i:o + 32 * i + 32], "little") for i in range(k)]
    A["r"], B["r"] = pts(lay["off_pa"], mA), pts(lay["off_pb"], d)
    return dict(A=A, B=B, proof=raw[:lay["la"] + lay["lb"]], point=pts(lay["off_pt"], d + n),
                claim=pts(lay["off_c"], 1)[0])


def relu_prove_chained_dev(ctx: Context, tr: Transcript, Z: torch.Tensor, GA: torch.Tensor, Q: int, R: int,
                           d_pts: torch.Tensor, range_flag: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_relu_prove_chained_dev: the zkReLU proof at given points (device canonical, 4 x logD)."""
    logD = _log2(Z.numel())
    n = relu_prove_len(logD, Q, R)
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=Z.device)
    assert out.dtype == torch.uint8 and out.numel() >= n and out.is_contiguous()
    assert d_pts.numel() == 128 * logD
    ln = ctypes.c_uint64(out.numel())
    ctx.check(lib().zk_relu_prove_chained_dev(ctx.h, tr.h, _dev_ptr(Z, torch.int32), _dev_ptr(GA, torch.int32), logD, Q, R,
                                              _dev_ptr(d_pts, torch.uint8), out.data_ptr(), ctypes.byref(ln),
                                              range_flag.data_ptr()))
    return out


# ---------------------------------------------------------------- N2: the top layer (D24, D26)
def loss_grad_prove_dev(ctx: Context, tr: Transcript, GZ: torch.Tensor, Z: torch.Tensor, Y: torch.Tensor,
                        out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_loss_grad_prove_dev: out = u (m canonical) | G_Z~(u), Z~(u), Y~(u) (canonical); asynchronous."""
    m = _log2(Z.numel())
    n = 32 * m + 96
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=Z.device)
    ln = ctypes.c_uint64(out.numel())
    ctx.check(lib().zk_loss_grad_prove_dev(ctx.h, tr.h, _dev_ptr(GZ, torch.int32), _dev_ptr(Z, torch.int32),
                                           _dev_ptr(Y, torch.int32), m, out.data_ptr(), ctypes.byref(ln)))
    return out


def rescale_prove_len(logD: int, Q: int, R: int) -> int:
    m = relu_logB(Q, R) + logD
    return _a16(12 + 64 + 2 * (12 + 32 + 96 * m + 64)) + 64 * m


def rescale_prove_dev(ctx: Context, tr: Transcript, Z: torch.Tensor, Q: int, R: int, d_pts: torch.Tensor,
                      range_flag: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_rescale_prove_dev (D26) at the points d_pts (device canonical: u_Z then u_P)."""
    logD = _log2(Z.numel())
    n = rescale_prove_len(logD, Q, R)
    if out is None:
        out = torch.empty(n, dtype=torch.uint8, device=Z.device)
    assert d_pts.numel() == 64 * logD
    ln = ctypes.c_uint64(out.numel())
    ctx.check(lib().zk_rescale_prove_dev(ctx.h, tr.h, _dev_ptr(Z, torch.int32), logD, Q, R, _dev_ptr(d_pts, torch.uint8),
                                         out.data_ptr(), ctypes.byref(ln), range_flag.data_ptr()))
    return out


def parse_rescale_out(raw: bytes, logD: int, Q: int, R: int) -> dict:
    m = relu_logB(Q, R) + logD
    lp = 12 + 32 + 96 * m + 64
    plen = 12 + 64 + 2 * lp
    A, B = parse_sumcheck_proof(raw[76:76 + lp]), parse_sumcheck_proof(raw[76 + lp:plen])
    o = _a16(plen)
    A["r"] = [int.from_bytes(raw[o + 32 * i:o + 32 * i + 32], "little") for i in range(m)]
    B["r"] = [int.from_bytes(raw[o + 32 * (m + i):o + 32 * (m + i) + 32], "little") for i in range(m)]
    claims = [int.from_bytes(raw[12 + 32 * i:44 + 32 * i], "little") for i in range(2)]
    return dict(claims=claims, A=A, B=B, proof=raw[:plen])


def undelta_i8(ctx: Context, base16: torch.Tensor, delta8: torch.Tensor | None, L: int, n_slots: int,
               out: torch.Tensor) -> torch.Tensor:
    """zk_undelta_i8: base16 [L][...] int16 and delta8 [n_slots - L][...] int8 device tensors -> out[:n_slots] int32
    (out[s] = base[s], s < L; out[s] = out[s - L] + delta[s - L]), on the context stream."""
    assert base16.dtype == torch.int16 and base16.is_cuda and base16.is_contiguous() and base16.shape[0] == L
    slot = base16[0].numel()
    if delta8 is not None:
        assert delta8.dtype == torch.int8 and delta8.is_contiguous() and delta8.shape[0] == n_slots - L
    assert out.dtype == torch.int32 and out.is_contiguous() and out[0].numel() == slot
    ctx.check(lib().zk_undelta_i8(ctx.h, base16.data_ptr(), delta8.data_ptr() if delta8 is not None else None, slot, L,
                                  n_slots, out.data_ptr()))
    return out


def widen_i16(ctx: Context, t16: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """zk_widen_i16: an int16 device tensor -> int32 (same shape), on the context stream."""
    assert t16.dtype == torch.int16 and t16.is_cuda and t16.is_contiguous()
    if out is None:
        out = torch.empty(t16.shape, dtype=torch.int32, device=t16.device)
    ctx.check(lib().zk_widen_i16(ctx.h, t16.data_ptr(), t16.numel(), out.data_ptr()))
    return out
