"""FAC4DNN family driver (PAPER Example 2 P:L292-312, Protocol 1 line 7 P:L326).

Fiat-Shamir per proving window (D3d): the window transcript absorbs "fcn/hdr",
then for every family in the fixed order of synth.fcn.assemble_families
"fcn/fam" <name> and forks the family's own transcript, on which the family's
protocol runs — matmul families: zk_matmul_prove (the
reduction of zk_matmul_reduce then zk_sumcheck_prove with m = logN + logD2,
n_eq = logN, K = 2); ReLU families: zk_relu_prove_dev.  Stack tensors must
already be resident on the device; this module only sequences the library calls
(no arithmetic here).  The window absorbs every family's final state at the end
("fcn/join").  Independent transcripts let the zkReLU family run on a second
stream concurrently with the matmul families.  Every family writes into one
device buffer and the window synchronises once, when the proofs are copied back.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import api


@dataclass
class DeviceFamily:
    name: str
    kind: str                  # "matmul" | "relu"
    A: torch.Tensor = None
    B: torch.Tensor = None
    trans_a: bool = False
    trans_b: bool = False
    Z: torch.Tensor = None
    GA: torch.Tensor = None
    Q: int = 16
    R: int = 16


def upload_families(families, device="cuda", pin: bool = False) -> list:
    """Copy synth.fcn families (numpy int32 stacks) to the device; a stack shared by several
    families (same array) is copied once and shared."""
    out = []
    seen = {}

    def dev(a):
        if id(a) not in seen:
            t = torch.from_numpy(a)
            if pin:
                t = t.pin_memory()
            seen[id(a)] = t.to(device, non_blocking=pin)
        return seen[id(a)]

    for f in families:
        if hasattr(f, "A"):
            out.append(DeviceFamily(f.name, "matmul", A=dev(f.A), B=dev(f.B), trans_a=f.transA, trans_b=f.transB))
        else:
            out.append(DeviceFamily(f.name, "relu", Z=dev(f.Z), GA=dev(f.GA), Q=f.Q, R=f.R))
    return out


def _layout(f: DeviceFamily, merge_aux: bool = False):
    if f.kind == "matmul":
        logs = api._mm_logs(f.A, f.B, f.trans_a, f.trans_b)
        return logs, api.matmul_prove_len(logs)
    logD = api._log2(f.Z.numel())
    n = api.relu_prove_len(logD, f.Q, f.R)
    if merge_aux:   # the aux-claim merge output follows at the next 16-byte offset
        n = api._a16(n) + api.relu_merge_len(f.Q, f.R)
    return logD, n


def _slot(n: int) -> int:
    return (n + 32 + 255) & ~255   # family output + 32-byte state, every family 256-byte aligned


def window_out_bytes(families: list, merge_aux: bool = False) -> int:
    """Size of a window's device output buffer (what collect_window copies back)."""
    return sum(_slot(_layout(f, merge_aux)[1]) for f in families) + 256   # + the window's final state


def _family_work(f: DeviceFamily) -> int:
    if f.kind == "matmul":
        return f.A.numel() + f.B.numel()
    return 64 * f.Z.numel()


def enqueue_window(ctx: api.Context, seed: bytes, header: bytes, families: list, ready: list | None = None,
                   relu_ctx: api.Context | None = None, proof_order: list | None = None,
                   mm_ctxs: list | None = None, merge_aux: bool = False, wctx: api.Context | None = None):
    """Enqueue one window's proofs without synchronising.

    Transcripts (D3d): the window transcript W absorbs "fcn/hdr", then per family "fcn/fam"
    <name> and forks that family's transcript ("fcn/fork"); every family is proved on its own
    transcript; W finally absorbs "fcn/join" <family state> for every family.  With relu_ctx (a context
    on a second stream) the zkReLU families run there, concurrently with the matmul families on ctx.
    ready (optional): one torch.cuda.Event per family that its stream waits on before its proof (the
    end of its host->device upload on a copy stream).  proof_order (optional): the order in which the
    families' proofs are enqueued (indices into `families`); forks and joins always follow the list
    order, so the transcripts and proof bytes do not depend on it.
    mm_ctxs (optional): extra contexts (own streams, typically with an SM budget) over which the matmul
    families are spread, largest first onto the least-loaded one, so their latency-bound sumchecks run
    side by side; ctx keeps its share.
    wctx (optional): the context of the window transcript W (default ctx).  With a wctx of its own per
    window (alternating), nothing in a window waits for the previous window's families, so windows
    enqueued back to back pipeline (a window's latency-bound tail overlaps the next one's rounds); the
    child transcripts are then released by collect_window.
    Returns (out, flag, layout): `out` holds, per family, its proof output followed by the family
    transcript's final state, then W's final state; `flag` is the int32 range flag."""
    dev = (families[0].A if families[0].kind == "matmul" else families[0].Z).device
    lay = []
    off = 0
    for f in families:
        info, n = _layout(f, merge_aux)
        lay.append((f, info, off, n))
        off += _slot(n)
    two = relu_ctx is not None and relu_ctx.stream != ctx.stream
    lanes = [ctx] + [c for c in (mm_ctxs or []) if c.stream != ctx.stream]
    home = {}
    load = [0] * len(lanes)
    for i in sorted(range(len(families)), key=lambda i: -_family_work(families[i])):
        if families[i].kind == "matmul":
            j = min(range(len(lanes)), key=lambda j: load[j])
            home[i] = lanes[j]
            load[j] += _family_work(families[i])
    ctx_of_i = lambda i: relu_ctx if (two and families[i].kind == "relu") else home.get(i, ctx)
    own_w = wctx is not None and wctx.stream != ctx.stream
    wc = wctx if own_w else ctx
    # streams that fork from and join back into the window transcript's stream
    side = ([relu_ctx] if two else []) + (lanes if own_w else lanes[1:])
    # the output buffer and the range flag on the window transcript's stream: every proof stream forks from
    # it after the zero fill, whatever the caller's current stream is
    with torch.cuda.stream(wc.stream):
        out = torch.empty(off + 256, dtype=torch.uint8, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    W = api.Transcript(wc, seed)
    W.absorb("fcn/hdr", header)
    kids = []
    for i, f in enumerate(families):
        W.absorb("fcn/fam", f.name.encode())
        kids.append(W.fork("fcn/fork", ctx_of_i(i)))
    if side:
        ev = torch.cuda.Event()
        ev.record(wc.stream)
        for c in side:
            c.stream.wait_event(ev)
    for i in (proof_order if proof_order is not None else range(len(lay))):
        f, info, o, n = lay[i]
        c, T = ctx_of_i(i), kids[i]
        if ready is not None:
            c.stream.wait_event(ready[i])
        if f.kind == "matmul":
            api.matmul_prove(c, T, f.A, f.B, f.trans_a, f.trans_b, out=out[o:o + n])
        else:
            rn = api.relu_prove_len(info, f.Q, f.R)
            api.relu_prove_dev(c, T, f.Z, f.GA, f.Q, f.R, flag, out=out[o:o + rn])
            if merge_aux:
                mo = o + api._a16(rn)
                api.relu_merge_dev(c, T, f.Z, f.GA, f.Q, f.R, out[o:o + rn], out=out[mo:o + n])
        T.state_dev(out[o + n:o + n + 32])
    for c in side:
        ev = torch.cuda.Event()
        ev.record(c.stream)
        wc.stream.wait_event(ev)
    for T in kids:
        W.absorb_state("fcn/join", T)
    W.state_dev(out[off:off + 32])
    if own_w:   # pipelined windows: the transcripts are released by collect_window, after the device work
        lay.append(("transcripts", kids + [W]))
        return out, flag, lay
    if side:   # the children are freed on their own streams: after the joins
        ev = torch.cuda.Event()
        ev.record(ctx.stream)
        for c in side:
            c.stream.wait_event(ev)
    for T in kids:
        T.close()
    W.close()   # stream-ordered: the state buffers are released after the enqueued work
    return out, flag, lay


def collect_window(out: torch.Tensor, flag: torch.Tensor, lay) -> list:
    """Copy a window's outputs to the host (the one synchronisation) and parse them.  The last result
    also carries "window_state" (the window transcript after the joins)."""
    torch.cuda.synchronize(out.device)   # the library wrote on its contexts' streams
    raw = out.cpu().numpy().tobytes()
    if lay and lay[-1][0] == "transcripts":
        for T in lay[-1][1]:
            T.close()
        lay = lay[:-1]
    if int(flag.item()) & 1:
        raise api.ZkError(-2, "zkReLU input outside the (Q+R)-bit range")
    results = []
    for f, info, o, n in lay:
        blob = raw[o:o + n]
        if f.kind == "matmul":
            r = api.parse_matmul_out(blob, info)
            res = dict(name=f.name, kind="matmul", w=r["w"], u1=r["u1"], u3=r["u3"], claim=r["claim"],
                       msgs=r["msgs"], r=r["r"], finals=r["finals"], proof=r["proof"])
        else:
            rn = api.relu_prove_len(info, f.Q, f.R)
            r = api.parse_relu_out(blob[:rn], info, f.Q, f.R)
            res = dict(name=f.name, kind="relu", claims=r["claims"], msgs=r["msgs"], point=r["point"],
                       finals=r["finals"], proof=r["proof"])
            if len(blob) > rn:
                res["merge"] = api.parse_relu_merge_out(blob[api._a16(rn):], f.Q, f.R)
        res["state"] = raw[o + n:o + n + 32]
        results.append(res)
    end = len(raw) - 256
    results[-1]["window_state"] = raw[end:end + 32]
    return results


def prove_window(ctx: api.Context, seed: bytes, header: bytes, families: list,
                 relu_ctx: api.Context | None = None, mm_ctxs: list | None = None, merge_aux: bool = False) -> list:
    """Prove every family of one window (D3d transcripts); returns per-family results."""
    return collect_window(*enqueue_window(ctx, seed, header, families, relu_ctx=relu_ctx, mm_ctxs=mm_ctxs,
                                          merge_aux=merge_aux))


class HostStack:
    """A host stack whose trailing slots are zero padding (the stack axis padded to a power of two,
    P:L144): only the leading `data.shape[0]` slots travel over PCIe; the device tensor has `shape` and its
    padding slots are zero-filled on the device."""

    def __init__(self, data: torch.Tensor, shape):
        self.data, self.shape = data, tuple(shape)
        self.dtype = data.dtype

    def data_ptr(self) -> int:
        return self.data.data_ptr()

    def numel(self) -> int:
        return self.data.numel()

    def element_size(self) -> int:
        return self.data.element_size()


class DeltaStack:
    """A host stack shipped as its first L slots (int16) and the int8 differences of every later real slot to
    the slot L before it (a weight stack: the slot of the same layer one training step earlier); rebuilt on
    the device by zk_undelta_i8 into the int32 stack of `shape` (trailing padding slots zero-filled once).
    delta_stack() builds one when every difference fits int8 and the first slots fit int16."""

    def __init__(self, base: torch.Tensor, delta, L: int, n_real: int, shape):
        self.base, self.delta, self.L, self.n_real, self.shape = base, delta, int(L), int(n_real), tuple(shape)
        self.dtype = torch.int8

    def data_ptr(self) -> int:
        return self.base.data_ptr()

    def numel(self) -> int:   # the transport bytes (element_size 1)
        return self.base.numel() * 2 + (self.delta.numel() if self.delta is not None else 0)

    def element_size(self) -> int:
        return 1


def delta_stack(a, n_real: int, max_stride: int = 16, pin: bool = True):
    """numpy int32 stack a[N][...] (slots >= n_real zero padding) -> DeltaStack with the smallest stride L <=
    max_stride for which a[s] - a[s - L] fits int8 for every real slot s >= L (and a[:L] fits int16), else None.
    Transport encoding only: the device rebuilds a[:n_real] exactly."""
    import numpy as np
    body = a[:n_real]
    if a.ndim < 2 or n_real < 2 or body[0].size % 4:
        return None
    for L in range(1, min(max_stride, n_real - 1) + 1):
        base = body[:L]
        if int(base.max()) >= (1 << 15) or int(base.min()) < -(1 << 15):
            return None
        d = body[L:].astype(np.int64) - body[:-L]
        if int(d.max()) <= 127 and int(d.min()) >= -128:
            tb = torch.from_numpy(np.ascontiguousarray(base.astype(np.int16)))
            td = torch.from_numpy(np.ascontiguousarray(d.astype(np.int8)))
            if pin:
                tb, td = tb.pin_memory(), td.pin_memory()
            return DeltaStack(tb, td, L, n_real, a.shape)
    return None


_RING: dict = {}   # persistent transport buffers: (device, host buffer, window slot) -> (staging, int32 output)


def release_transport_buffers() -> None:
    """Free the persistent device buffers of the end-to-end transport (prove_window(s)_from_host)."""
    _RING.clear()


class _Uploader:
    """Host stacks -> int32 device tensors.  The copy stream `cs` carries only the host->device DMA, so the
    copy engine streams without gaps; the device-side work of an upload (widening an int16 stack,
    zk_widen_i16) runs on a second stream `ws` behind an event per copy.  (On one stream a widen kernel
    queued behind a long proof kernel holding every SM stalled the DMA of all later stacks.)  With a window
    `slot` the staging and int32 buffers are persistent (allocated once per host stack and slot, a
    HostStack's padding slots zero-filled once): the caching allocator's cudaMalloc calls and their
    synchronisation stay out of the transport (uploads of the C4 window 10.8-13.5 -> ~8.7 ms, the DMA
    time).  ready() gives an event after every upload enqueued so far."""

    def __init__(self, dev, cs):
        self.dev, self.cs = dev, cs
        self.ws = torch.cuda.Stream(device=dev)
        self.wctx = api.Context(dev.index if dev.index is not None else torch.cuda.current_device(), self.ws)

    def _delta_buffers(self, t, slot):
        key = (self.dev.index, t.base.data_ptr(), t.numel(), "delta", t.shape, slot)
        bufs = _RING.get(key) if slot is not None else None
        if bufs is None:
            with torch.cuda.stream(self.cs):
                sb = torch.empty(tuple(t.base.shape), dtype=torch.int16, device=self.dev)
                sd = torch.empty(tuple(t.delta.shape), dtype=torch.int8, device=self.dev) if t.delta is not None else None
                out = torch.empty(t.shape, dtype=torch.int32, device=self.dev)
                if t.n_real < t.shape[0]:
                    out[t.n_real:].zero_()
            bufs = (sb, sd, out)
            if slot is not None:
                _RING[key] = bufs
        return bufs

    def _buffers(self, t, slot):
        hs = isinstance(t, HostStack)
        data = t.data if hs else t
        shape = t.shape if hs else tuple(data.shape)
        key = (self.dev.index, data.data_ptr(), data.numel(), data.dtype, shape, slot)
        bufs = _RING.get(key) if slot is not None else None
        if bufs is None:
            with torch.cuda.stream(self.cs):
                stage = torch.empty(tuple(data.shape), dtype=data.dtype, device=self.dev) \
                    if (hs or data.dtype != torch.int32) else None
                out = torch.empty(shape, dtype=torch.int32, device=self.dev)
                if data.shape[0] < shape[0]:
                    out[data.shape[0]:].zero_()
            bufs = (stage, out)
            if slot is not None:
                _RING[key] = bufs
        return data, bufs

    def upload(self, t, slot=None) -> torch.Tensor:
        if isinstance(t, DeltaStack):   # int16 first slots + int8 differences, rebuilt by zk_undelta_i8
            sb, sd, out = self._delta_buffers(t, slot)
            with torch.cuda.stream(self.cs):
                sb.copy_(t.base, non_blocking=True)
                if sd is not None:
                    sd.copy_(t.delta, non_blocking=True)
            self.ws.wait_stream(self.cs)
            with torch.cuda.stream(self.ws):
                api.undelta_i8(self.wctx, sb, sd, t.L, t.n_real, out)
            return out
        data, (stage, out) = self._buffers(t, slot)
        n = data.shape[0]
        if stage is None:   # int32 stack, no padding: the copy is the upload
            with torch.cuda.stream(self.cs):
                out.copy_(data, non_blocking=True)
            self.ws.wait_stream(self.cs)
            return out
        with torch.cuda.stream(self.cs):
            stage.copy_(data, non_blocking=True)
        self.ws.wait_stream(self.cs)
        with torch.cuda.stream(self.ws):
            if data.dtype == torch.int16:
                api.widen_i16(self.wctx, stage, out=out[:n])
            else:
                out[:n].copy_(stage)
        return out

    def ready(self) -> torch.cuda.Event:
        ev = torch.cuda.Event()
        ev.record(self.ws)
        return ev


def prove_window_from_host(ctx: api.Context, seed: bytes, header: bytes, host_families, copy_stream=None,
                           relu_ctx: api.Context | None = None, mm_ctxs: list | None = None,
                           merge_aux: bool = False) -> list:
    """The user-facing end-to-end call: families given as host (ideally pinned) int32 tensors.

    Each family's stacks are copied host->device on `copy_stream` (one is created if None) and its
    proof waits only for its own upload, so the transfers of later families overlap the proofs of
    earlier ones.  A host buffer shared by several families (the weight stack W[2..8] is the B operand
    of F[2..8] and of GA[1..7]) is copied once.  The proof bytes come back to the host (one
    synchronisation).  host_families: DeviceFamily records whose tensors live on the host (int32, or int16
    for stacks whose entries fit 16 bits: copied as int16 and widened on the device, zk_widen_i16)."""
    dev = torch.device("cuda", ctx.device)
    cs = copy_stream if copy_stream is not None else torch.cuda.Stream(device=dev)
    up_ = _Uploader(dev, cs)
    fams, ready = [], []
    uploaded = {}   # host buffer -> device tensor: a stack shared by several families is copied once

    def upload(t):
        key = (t.data_ptr(), t.numel(), t.dtype)
        if key not in uploaded:
            uploaded[key] = up_.upload(t, slot=0)
        return uploaded[key]

    # upload (and proof) order: zkReLU families first (least data, most work), then the matmul
    # families by decreasing operand bytes, so the families proved last have the least left to do
    def nbytes(f):
        ts = (f.A, f.B) if f.kind == "matmul" else (f.Z, f.GA)
        return sum(t.numel() * t.element_size() for t in ts)
    order = sorted(range(len(host_families)),
                   key=lambda i: (host_families[i].kind != "relu", -nbytes(host_families[i]), i))
    fams, ready = [None] * len(host_families), [None] * len(host_families)
    for i in order:
        f = host_families[i]
        up = {k: upload(getattr(f, k)) for k in (("A", "B") if f.kind == "matmul" else ("Z", "GA"))}
        g = DeviceFamily(f.name, f.kind, trans_a=f.trans_a, trans_b=f.trans_b, Q=f.Q, R=f.R, **up)
        readers = [relu_ctx.stream] if (relu_ctx is not None and f.kind == "relu") else \
            [ctx.stream] + [c.stream for c in (mm_ctxs or [])]
        for t in up.values():   # the proof reads it on its family's stream
            for st in readers:
                t.record_stream(st)
        fams[i] = g
        ready[i] = up_.ready()
    return collect_window(*enqueue_window(ctx, seed, header, fams, ready, relu_ctx=relu_ctx, proof_order=order,
                                          mm_ctxs=mm_ctxs, merge_aux=merge_aux))


def upload_windows(windows: list, copy_stream=None, device: int = 0) -> list:
    """The uploads of prove_windows_from_host alone (diagnostics: the end-to-end leg's transport time)."""
    dev = torch.device("cuda", device)
    cs = copy_stream if copy_stream is not None else torch.cuda.Stream(device=dev)
    up_ = _Uploader(dev, cs)
    out = []
    for w, host_families in enumerate(windows):
        uploaded = {}
        for f in host_families:
            for k in (("A", "B") if f.kind == "matmul" else ("Z", "GA")):
                t = getattr(f, k)
                key = (t.data_ptr(), t.numel(), t.dtype)
                if key not in uploaded:
                    uploaded[key] = up_.upload(t, slot=w)
        out.append(uploaded)
    torch.cuda.current_stream(dev).wait_stream(up_.ws)
    return out


def prove_windows_from_host(ctx: api.Context, windows: list, copy_stream=None, relu_ctx: api.Context | None = None,
                            mm_ctxs: list | None = None, merge_aux: bool = False) -> list:
    """Several windows end to end, pipelined: windows = [(seed, header, host_families), ...].  Every
    window's uploads are enqueued on the copy stream behind the previous window's, and its proofs wait
    only for their own uploads, so the copy engine streams without gaps while earlier windows prove;
    the proofs of all windows come back with one synchronisation at the end.  Same bytes as
    prove_window_from_host per window."""
    dev = torch.device("cuda", ctx.device)
    cs = copy_stream if copy_stream is not None else torch.cuda.Stream(device=dev)
    up_ = _Uploader(dev, cs)
    pending = []
    for w, (seed, header, host_families) in enumerate(windows):
        uploaded = {}

        def upload(t, w=w):
            key = (t.data_ptr(), t.numel(), t.dtype)
            if key not in uploaded:
                uploaded[key] = up_.upload(t, slot=w)
            return uploaded[key]

        def nbytes(f):
            ts = (f.A, f.B) if f.kind == "matmul" else (f.Z, f.GA)
            return sum(t.numel() * t.element_size() for t in ts)
        order = sorted(range(len(host_families)),
                       key=lambda i: (host_families[i].kind != "relu", -nbytes(host_families[i]), i))
        fams, ready = [None] * len(host_families), [None] * len(host_families)
        for i in order:
            f = host_families[i]
            up = {k: upload(getattr(f, k)) for k in (("A", "B") if f.kind == "matmul" else ("Z", "GA"))}
            fams[i] = DeviceFamily(f.name, f.kind, trans_a=f.trans_a, trans_b=f.trans_b, Q=f.Q, R=f.R, **up)
            readers = [relu_ctx.stream] if (relu_ctx is not None and f.kind == "relu") else \
                [ctx.stream] + [c.stream for c in (mm_ctxs or [])]
            for t in up.values():
                for st in readers:
                    t.record_stream(st)
            ready[i] = up_.ready()
        pending.append(enqueue_window(ctx, seed, header, fams, ready, relu_ctx=relu_ctx, proof_order=order,
                                      mm_ctxs=mm_ctxs, merge_aux=merge_aux))
    return [collect_window(*p) for p in pending]
