"""The claim-chained FAC4DNN window on the device (Protocol 1 lines 7-8, P:L320-333;
DESIGN.md D25).  Sequencing of library calls only (no arithmetic here).

Window transcript W ("fcn/chdr" header), three stages, each a set of forked transcripts joined back:
  1. every matmul family (zk_matmul_prove on its fork, spread over the matmul streams) and the loss family
     (zk_loss_grad_prove_dev, D24);
  2. every tensor family whose claims need merging (zk_claim_merge_dev: the claims of stage 1 on views of
     it -> one claim on its stack), spread over all streams;
  3. every ReLU family: zk_relu_prove_chained_dev at the merged points of its Z, A, G_A, G_Z stacks
     (P:L186), then the aux-claim merge (zk_relu_merge_dev, D21); the top layer's rescale
     (zk_rescale_prove_dev, D26) at the claims on Z^(L) and Z^(L)', then the merge of its two aux claims.
The window ends with one claim per committed tensor family and one on each aux (verify.verify_window_chained
returns exactly those).  The claims of stage 1 travel to stage 2 as device bytes (slices of the window's
output buffer gathered on the consuming stream), so the whole window is one stream-ordered program with
a single host synchronisation.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import api
from .fcn import DeviceFamily
from .plan import RELU_ROLES, family_kind, is_whole, matmul_claim_pieces


@dataclass
class DeviceTensor:
    """A tensor family on the device: N slots of rows x cols int32 (pad[j]: slot j is zero padding);
    committed ones hold their stack, ReLU-bound ones name the ReLU family whose words they are formed from."""
    name: str
    kind: str
    pad: list
    rows: int
    cols: int
    relu: str | None = None
    array: torch.Tensor | None = None


@dataclass
class ChainedFamily(DeviceFamily):
    refs: dict = field(default_factory=dict)      # matmul / loss: role -> (tensor name, map)
    tensors: dict = field(default_factory=dict)   # ReLU / rescale: role -> tensor name
    GZ: torch.Tensor = None                       # loss family (D24): G_Z^(L), Z^(L)', Y stacks
    Zp: torch.Tensor = None
    Y: torch.Tensor = None


def upload_plan(families, tensors, device="cuda", top=None) -> tuple:
    """synth.fcn families + plan_window tensor families -> device records; an array shared by several
    families or tensor families (same numpy object) is copied once."""
    seen = {}

    def dev(a):
        if id(a) not in seen:
            seen[id(a)] = torch.from_numpy(a).to(device)
        return seen[id(a)]

    fams = []
    for f in list(families) + list(top or []):
        k = family_kind(f)
        if k == "matmul":
            fams.append(ChainedFamily(f.name, "matmul", A=dev(f.A), B=dev(f.B), trans_a=f.transA, trans_b=f.transB,
                                      refs={k: (r.tensor, list(r.map)) for k, r in f.refs.items()}))
        elif k == "loss":
            fams.append(ChainedFamily(f.name, "loss", GZ=dev(f.GZ), Zp=dev(f.Zp), Y=dev(f.Y),
                                      refs={k: (r.tensor, list(r.map)) for k, r in f.refs.items()}))
        elif k == "rescale":
            fams.append(ChainedFamily(f.name, "rescale", Z=dev(f.Z), Q=f.Q, R=f.R, tensors=dict(f.tensors)))
        else:
            fams.append(ChainedFamily(f.name, "relu", Z=dev(f.Z), GA=dev(f.GA), Q=f.Q, R=f.R, tensors=dict(f.tensors)))
    ts = [DeviceTensor(t.name, t.kind, [s is None for s in t.slots], t.rows, t.cols, t.relu,
                       None if t.array is None else dev(t.array)) for t in tensors]
    return fams, ts


def _slot(n: int) -> int:
    return (n + 32 + 255) & ~255


def _log2(n: int) -> int:
    return api._log2(n)


def _mm_pieces(logs) -> dict:
    """Byte ranges (offset, elements) of the named pieces in a zk_matmul_prove output."""
    lN, l1, l2, l3 = logs
    np_, m = lN + l1 + l3, lN + l2
    off = 32 * np_ + 32
    plen = 12 + 32 + 96 * m + 64
    o_r = api._a16(off + plen)
    return dict(w=(0, lN), u1=(32 * lN, l1), u3=(32 * (lN + l1), l3), claim=(32 * np_, 1),
                fA=(off + plen - 64, 1), fB=(off + plen - 32, 1), rn=(o_r, lN), rk=(o_r + 32 * lN, l2))


class _Lanes:
    """Streams a stage spreads its proofs over (least-loaded first)."""

    def __init__(self, ctxs):
        self.ctxs, self.load = ctxs, [0] * len(ctxs)

    def pick(self, work: int):
        j = min(range(len(self.ctxs)), key=lambda j: self.load[j])
        self.load[j] += work
        return self.ctxs[j]


def _fence(src, dsts):
    ev = torch.cuda.Event()
    ev.record(src.stream)
    for c in dsts:
        if c.stream != src.stream:
            c.stream.wait_event(ev)


def enqueue_window_chained(ctx: api.Context, seed: bytes, header: bytes, families: list, tensors: list,
                           relu_ctx: api.Context | None = None, mm_ctxs: list | None = None,
                           wctx: api.Context | None = None, merge_ctxs: list | None = None, serial: bool = False,
                           marks: list | None = None, rescale_ctx: api.Context | None = None,
                           late_ctxs: list | None = None, late_after_relu: bool = False):
    """Enqueue one chained window without synchronising; returns a handle for collect_window_chained.
    Streams: the window transcript W on wctx (default ctx); stages 1-2 over ctx + mm_ctxs; stage 3 on
    relu_ctx.  Nothing at the end of a window makes the stage 1-2 streams wait for its stage 3 (the
    child transcripts are freed in collect_window_chained), so with a different wctx per window the
    next window's matmul families and merges run while this window's zkReLU proves.  merge_ctxs
    (optional): the streams stage 2 spreads its claim merges over (latency-bound sumchecks: many
    budgeted streams side by side), default ctx + mm_ctxs.  serial: the window starts after the zkReLU stream's
    earlier work (no overlap with the previous window's stage 3).  rescale_ctx (optional): the stream of the
    top layer's rescale and its aux merge, which then run beside the zkReLU instead of after it (their
    transcript is a fork of its own, so only the scheduling changes, not a byte of the window).  late_ctxs
    (optional): the streams of the claim merges stage 3 does not wait for (D25 order: forked after stage 3's
    families), which then prove beside the zkReLU; default the zkReLU's stream (after it).  late_after_relu:
    the late merges and the rescale start when the zkReLU sumcheck has been proved (beside its aux merge),
    not at the start of stage 3 (the zkReLU's single-wave kernels lose most to throughput work beside them).  Co-residency:
    k_relu_ipersist (129 CTAs, two per SM) must always find its SMs next to the persistent sumcheck grids
    (k_sc_all, one SM per CTA) of the streams that run beside it, so the SM budgets of rescale_ctx and
    late_ctxs should add up to <= 148 - 65.  marks (diagnostics): a list that receives
    (label, stream, timing event) at the window's start, after every family / merge and at each stage join."""

    def mark(label, c):
        if marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(c.stream)
            marks.append((label, c.stream, ev))
    dev = next(f.A for f in families if f.kind == "matmul").device
    mms = [f for f in families if f.kind == "matmul"]
    losses = [f for f in families if f.kind == "loss"]
    relus = [f for f in families if f.kind == "relu"]
    rescales = [f for f in families if f.kind == "rescale"]
    tmap = {t.name: t for t in tensors}
    lanes1 = [ctx] + [c for c in (mm_ctxs or []) if c.stream != ctx.stream]
    rctx = relu_ctx if relu_ctx is not None else ctx
    sctx = rescale_ctx if rescale_ctx is not None else rctx
    ctx3 = [rctx] + ([sctx] if sctx.stream != rctx.stream else [])
    lanes2b = list(late_ctxs) if late_ctxs else [rctx]
    ctx3 += [c for c in lanes2b if c.stream not in [x.stream for x in ctx3]]
    wctx = wctx if wctx is not None else ctx
    lanes2 = list(merge_ctxs) if merge_ctxs else lanes1
    # ---- layout of the window's output buffer
    off = 0
    lay1 = []
    for f in mms:
        logs = api._mm_logs(f.A, f.B, f.trans_a, f.trans_b)
        n = api.matmul_prove_len(logs)
        lay1.append((f, logs, off, n))
        off += _slot(n)
    layL = []
    for f in losses:
        m = _log2(f.GZ.numel())
        layL.append((f, m, off, 32 * m + 96))
        off += _slot(32 * m + 96)
    # the claims stage 1 leaves, per tensor family (in family order, roles Y, A, B; then G_Z, Z', Y)
    claims = {t.name: [] for t in tensors}
    for f, logs, o, n in lay1:
        pieces = _mm_pieces(logs)
        for role, vp, up, cp in matmul_claim_pieces(f.trans_a, f.trans_b):
            tname, mp = f.refs[role]
            rng = lambda names: [(o + pieces[p][0], pieces[p][1]) for p in names]
            claims[tname].append(dict(map=mp, v=rng(vp), u=rng(up), c=rng([cp]), src=(f.name, role)))
    for f, m, o, n in layL:
        d = _log2(f.GZ.shape[1] * f.GZ.shape[2])
        for k, role in enumerate(("GZ", "Zp", "Y")):
            tname, mp = f.refs[role]
            claims[tname].append(dict(map=mp, v=[(o, d)], u=[(o + 32 * d, m - d)], c=[(o + 32 * m + 32 * k, 1)],
                                      src=(f.name, role)))
    merges = [t for t in tensors if claims[t.name] and not is_whole(t.pad, [c["map"] for c in claims[t.name]])]
    # D25 order: the merges of the stacks stage 3 is bound to first (joined before stage 3), the others after
    # stage 3's forks
    bound = {f.tensors[k] for f in relus for k in RELU_ROLES} | {f.tensors[k] for f in rescales for k in ("Z", "Zp")}
    merges = [t for t in merges if t.name in bound] + [t for t in merges if t.name not in bound]
    n2a = sum(1 for t in merges if t.name in bound)
    lay2 = []
    for t in merges:
        n = _log2(len(t.pad))
        cl = claims[t.name]
        L = api.claim_merge_layout(n, len(cl), _log2(t.rows) + _log2(t.cols))
        lay2.append((t, n, cl, off, L))
        off += _slot(L["total"])
    lay3 = []
    for f in relus:
        logD = _log2(f.Z.numel())
        rn = api.relu_prove_len(logD, f.Q, f.R)
        n = api._a16(rn) + api.relu_merge_len(f.Q, f.R)
        lay3.append((f, logD, rn, off, n))
        off += _slot(n)
    layR = []
    for f in rescales:
        logD = _log2(f.Z.numel())
        logB = api.relu_logB(f.Q, f.R)
        rl = api.rescale_prove_len(logD, f.Q, f.R)
        L = api.claim_merge_layout(0, 2, logD + logB)
        layR.append((f, logD, logB, rl, L, off, api._a16(rl) + L["total"]))
        off += _slot(api._a16(rl) + L["total"])
    with torch.cuda.stream(wctx.stream):   # on the window transcript's stream, which every stage forks from
        out = torch.empty(off + 256, dtype=torch.uint8, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    keep = []   # device temporaries in use by enqueued work

    def gather(c, ranges):
        with torch.cuda.stream(c.stream):
            g = torch.cat([out[a:a + 32 * k] for a, k in ranges if k]) if any(k for _, k in ranges) else \
                torch.zeros(0, dtype=torch.uint8, device=dev)
        keep.append(g)
        return g

    if serial:
        for c in ctx3:
            _fence(c, lanes1 + [wctx])
    W = api.Transcript(wctx, seed)
    mark("start", wctx)
    W.absorb("fcn/chdr", header)
    # ---- stage 1: the matmul families
    L1 = _Lanes(lanes1)
    home1 = {}
    for i in sorted(range(len(mms)), key=lambda i: -(mms[i].A.numel() + mms[i].B.numel())):
        home1[i] = L1.pick(mms[i].A.numel() + mms[i].B.numel())
    for i in range(len(losses)):
        home1[len(mms) + i] = L1.pick(losses[i].GZ.numel() * 3)
    kids1 = []
    for i, f in enumerate(mms + losses):
        W.absorb("fcn/fam", f.name.encode())
        kids1.append(W.fork("fcn/fork", home1[i]))
    _fence(wctx, lanes1)
    for i, (f, logs, o, n) in enumerate(lay1):
        c, T = home1[i], kids1[i]
        api.matmul_prove(c, T, f.A, f.B, f.trans_a, f.trans_b, out=out[o:o + n])
        T.state_dev(out[o + n:o + n + 32])
        mark("mm " + f.name, c)
    for i, (f, m, o, n) in enumerate(layL):
        c, T = home1[len(mms) + i], kids1[len(mms) + i]
        api.loss_grad_prove_dev(c, T, f.GZ, f.Zp, f.Y, out=out[o:o + n])
        T.state_dev(out[o + n:o + n + 32])
        mark("loss " + f.name, c)
    for c in lanes1:
        _fence(c, [wctx])
    for T in kids1:
        W.absorb_state("fcn/join", T)
    mark("stage 1 joined", wctx)
    # ---- stage 2: one claim per tensor family.  The merges wait for the zkReLU stream's earlier work (the
    # previous window's stage 3): their persistent grids and the zkReLU's persistent rounds (k_relu_ipersist,
    # ~65 SMs co-resident) then never compete for co-residency — measured, the overlapping version stalled
    # for tens to hundreds of milliseconds in some runs.  Stage 1 still overlaps the previous stage 3.
    for c3 in ctx3:
        if c3.stream not in [c.stream for c in lanes2]:
            _fence(c3, lanes2)
    lay2a, lay2b = lay2[:n2a], lay2[n2a:]
    L2 = _Lanes(lanes2)
    home2 = [L2.pick(len(t.pad) * t.rows * t.cols) for t, *_ in lay2a]
    kids2 = []
    for (t, *_), c in zip(lay2a, home2):
        W.absorb("fcn/tfam", t.name.encode())
        kids2.append(W.fork("fcn/fork", c))
    _fence(wctx, lanes2)

    def prove_merge(t, n, cl, o, L, c, T):
        d_pts = gather(c, [r for x in cl for r in x["v"] + x["u"]])
        d_cl = gather(c, [r for x in cl for r in x["c"]])
        maps = [x["map"] for x in cl]
        lr, lc = _log2(t.rows), _log2(t.cols)
        if t.array is not None:
            api.claim_merge_dev(c, T, t.array, n, lr, lc, maps, d_pts, d_cl, out=out[o:o + L["total"]])
        elif t.kind == "Zp":
            raise NotImplementedError("a claim merge on Z' (one loss claim on it is the whole stack)")
        else:
            f = next(g for g in relus if g.name == t.relu)
            src = {"Z": ("plain", f.Z, None), "GA": ("plain", f.GA, None), "A": ("relu_A", f.Z, None),
                   "GZ": ("relu_GZ", f.Z, f.GA)}[t.kind]
            api.claim_merge_dev(c, T, src[1], n, lr, lc, maps, d_pts, d_cl, source=src[0], X2=src[2], R=f.R,
                                out=out[o:o + L["total"]])
        T.state_dev(out[o + L["total"]:o + L["total"] + 32])
        mark("merge " + t.name, c)

    for (t, n, cl, o, L), c, T in zip(lay2a, home2, kids2):
        prove_merge(t, n, cl, o, L, c, T)
    for c in lanes2:
        _fence(c, [wctx])
    for T in kids2:
        W.absorb_state("fcn/join", T)
    mark("stage 2 joined", wctx)
    # ---- stage 3: the chained zkReLU families and their aux merges; the top layer's rescale
    pos2 = {t.name: (o, L) for t, n, cl, o, L in lay2}

    def point_ranges(tname):   # the one claim on a tensor family: its merge output, or its single claim
        if tname in pos2:
            to, tl = pos2[tname]
            d = _log2(tmap[tname].rows) + _log2(tmap[tname].cols)
            return [(to + tl["off_pt"], d + _log2(len(tmap[tname].pad)))]
        c0 = claims[tname][0]
        return c0["v"] + c0["u"]
    kids3 = []
    for f in relus + rescales:
        W.absorb("fcn/fam", f.name.encode())
        kids3.append(W.fork("fcn/fork", rctx if f.kind == "relu" else sctx))
    L2b = _Lanes(lanes2b)
    home2b = [L2b.pick(len(t.pad) * t.rows * t.cols) for t, *_ in lay2b]
    kids2b = []
    for (t, *_), c in zip(lay2b, home2b):
        W.absorb("fcn/tfam", t.name.encode())
        kids2b.append(W.fork("fcn/fork", c))
    _fence(wctx, ctx3)
    mark("stage 3 start", rctx)
    if late_ctxs and not late_after_relu:   # beside stage 3
        for (t, n, cl, o, L), c, T in zip(lay2b, home2b, kids2b):
            prove_merge(t, n, cl, o, L, c, T)
    for (f, logD, rn, o, n), T in zip(lay3, kids3):   # the zkReLU first: the window's critical path
        rngs = [r for role in RELU_ROLES for r in point_ranges(f.tensors[role])]
        d_pts = gather(rctx, rngs)
        api.relu_prove_chained_dev(rctx, T, f.Z, f.GA, f.Q, f.R, d_pts, flag, out=out[o:o + rn])
        mo = o + api._a16(rn)
        mark("relu proved " + f.name, rctx)
        if late_after_relu and f is relus[-1]:   # the late merges and the rescale beside the aux merge
            _fence(rctx, ([sctx] if sctx.stream != rctx.stream else []) + (lanes2b if late_ctxs else []))
            for (t, n_, cl, o_, L), c, T_ in zip(lay2b, home2b, kids2b):
                prove_merge(t, n_, cl, o_, L, c, T_)
        api.relu_merge_dev(rctx, T, f.Z, f.GA, f.Q, f.R, out[o:o + rn], out=out[mo:o + n])
        T.state_dev(out[o + n:o + n + 32])
        mark("relu+merge " + f.name, rctx)
    for (f, logD, logB, rl, L, o, n), T in zip(layR, kids3[len(relus):]):
        d_pts = gather(sctx, point_ranges(f.tensors["Z"]) + point_ranges(f.tensors["Zp"]))
        api.rescale_prove_dev(sctx, T, f.Z, f.Q, f.R, d_pts, flag, out=out[o:o + rl])
        # the two aux claims -> one (claim merge, D25, on the bits of Z: one slice [D][B])
        po = o + api._a16(12 + 64 + 2 * (12 + 32 + 96 * (logD + logB) + 64))
        pla = o + 76 + (12 + 32 + 96 * (logD + logB) + 64) - 32          # A's second final: aux~(r_A)
        plb = o + 76 + 2 * (12 + 32 + 96 * (logD + logB) + 64) - 64      # B's first final: aux~(r_B)
        d_apts = gather(sctx, [(po, logD + logB), (po + 32 * (logD + logB), logD + logB)])
        d_acl = gather(sctx, [(pla, 1), (plb, 1)])
        mo = o + api._a16(rl)
        api.claim_merge_dev(sctx, T, f.Z, 0, logD, logB, [[0], [0]], d_apts, d_acl, source="bits", R=f.Q + f.R,
                            out=out[mo:mo + L["total"]])
        T.state_dev(out[o + n:o + n + 32])
        mark("rescale+merge " + f.name, sctx)
    if not late_ctxs:   # after stage 3 on the zkReLU's stream
        for (t, n, cl, o, L), c, T in zip(lay2b, home2b, kids2b):
            prove_merge(t, n, cl, o, L, c, T)
    for c in ctx3:
        _fence(c, [wctx])
    for T in kids3 + kids2b:
        W.absorb_state("fcn/join", T)
    W.state_dev(out[off:off + 32])
    mark("end", wctx)
    return dict(out=out, flag=flag, lay1=lay1, layL=layL, lay2=lay2, lay3=lay3, layR=layR, end=off, keep=keep,
                claims=claims, transcripts=kids1 + kids2 + kids3 + kids2b + [W])


def collect_window_chained(h: dict) -> dict:
    """The one synchronisation: copy the window's outputs back and parse them.  Returns dict(matmul:
    name -> result, merges: tensor name -> result, relu: name -> result, window_state)."""
    torch.cuda.synchronize(h["out"].device)
    raw = h["out"].cpu().numpy().tobytes()
    for T in h.pop("transcripts", []):   # every use of the window's transcripts has completed
        T.close()
    if int(h["flag"].item()) & 1:
        raise api.ZkError(-2, "zkReLU input outside the (Q+R)-bit range")
    res = dict(matmul={}, merges={}, relu={}, loss={}, rescale={})
    for f, m, o, n in h["layL"]:
        vals = [int.from_bytes(raw[o + 32 * i:o + 32 * i + 32], "little") for i in range(m + 3)]
        res["loss"][f.name] = dict(u=vals[:m], claims=vals[m:], state=raw[o + n:o + n + 32])
    for f, logD, logB, rl, L, o, n in h["layR"]:
        am = api.parse_claim_merge_out(raw[o + api._a16(rl):o + api._a16(rl) + L["total"]], 0, 2, logD + logB)
        res["rescale"][f.name] = dict(proof=raw[o:o + 12 + 64 + 2 * (12 + 32 + 96 * (logD + logB) + 64)],
                                      aux_merge=am, state=raw[o + n:o + n + 32])
    for f, logs, o, n in h["lay1"]:
        r = api.parse_matmul_out(raw[o:o + n], logs)
        res["matmul"][f.name] = dict(logs=logs, w=r["w"], u1=r["u1"], u3=r["u3"], claim=r["claim"], msgs=r["msgs"],
                                     r=r["r"], finals=r["finals"], proof=r["proof"], state=raw[o + n:o + n + 32])
    for t, n, cl, o, L in h["lay2"]:
        d = _log2(t.rows) + _log2(t.cols)
        r = api.parse_claim_merge_out(raw[o:o + L["total"]], n, len(cl), d)
        r["state"] = raw[o + L["total"]:o + L["total"] + 32]
        res["merges"][t.name] = r
    for f, logD, rn, o, n in h["lay3"]:
        r = api.parse_relu_out(raw[o:o + rn], logD, f.Q, f.R)
        r["merge"] = api.parse_relu_merge_out(raw[o + api._a16(rn):o + n], f.Q, f.R)
        r["state"] = raw[o + n:o + n + 32]
        res["relu"][f.name] = r
    res["window_state"] = raw[h["end"]:h["end"] + 32]
    return res


def prove_window_chained(ctx: api.Context, seed: bytes, header: bytes, families: list, tensors: list,
                         relu_ctx: api.Context | None = None, mm_ctxs: list | None = None,
                         wctx: api.Context | None = None, merge_ctxs: list | None = None,
                         rescale_ctx: api.Context | None = None, late_ctxs: list | None = None,
                         late_after_relu: bool = False) -> dict:
    return collect_window_chained(enqueue_window_chained(ctx, seed, header, families, tensors, relu_ctx, mm_ctxs, wctx,
                                                         merge_ctxs, rescale_ctx=rescale_ctx, late_ctxs=late_ctxs,
                                                         late_after_relu=late_after_relu))
