"""Host verifiers (D23): ctypes marshalling of libzkdl's zk_verify_* /
zk_htr_* (verify.cu, plain host code), and the window verifier that replays the D3d fork/join
transcripts of a FAC4DNN proving window.

Verification replays the prover's rounds; every round identity and each protocol's final
identity is checked here.  The statement's shape is always the verifier's own (a proof whose header
differs is rejected before anything else is read).  Every value returned — claims, finals, points — is
read from the verified proof bytes or drawn by the verifier itself, never taken from the prover's
result dicts: those values are the claims left for the commitments (out of scope), so
a caller holding the tensors (tests) or their commitments closes them.
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


def _fin(proof: bytes, k: int) -> list:
    """The last k field elements of a proof (its finals), as bytes the verifier has just checked."""
    return [int.from_bytes(proof[len(proof) - 32 * (k - i):len(proof) - 32 * (k - i - 1)], "little") for i in range(k)]


def verify_sumcheck(tr: HostTranscript, proof: bytes, w: list, claim: int | None = None, *, shape) -> list:
    """zk_verify_sumcheck for the statement shape = (m, n_eq, K): returns the point r; raises Rejected."""
    m, n_eq, K = (int(v) for v in shape)
    if len(w) != n_eq:
        raise ValueError("w must have n_eq elements")
    pt = ctypes.create_string_buffer(32 * max(1, m))
    _run("sumcheck", lib().zk_verify_sumcheck, tr.st, proof, len(proof), (ctypes.c_uint32 * 3)(m, n_eq, K), _fr(w),
         None if claim is None else _fr([claim]), pt)
    return _ints(pt, m)


def sumcheck_finals(proof: bytes) -> list:
    K = int.from_bytes(proof[8:12], "little")
    return _fin(proof, K)


def verify_hadamard_zero(tr: HostTranscript, proof: bytes, m: int) -> dict:
    w, pt = ctypes.create_string_buffer(32 * max(1, m)), ctypes.create_string_buffer(32 * max(1, m))
    _run("hadamard zero", lib().zk_verify_hadamard_zero, tr.st, proof, len(proof), m, w, pt)
    return dict(w=_ints(w, m), r=_ints(pt, m), finals=_fin(proof, 3))


def relu_points(tr: HostTranscript, logD: int, Q: int, R: int) -> list:
    """The four points D3b draws (u_Z, u_A, u_GA, u_GZ) — drawn on a copy of the transcript."""
    T = HostTranscript(state=tr.state())
    T.absorb("relu/hdr", b"".join(int(v).to_bytes(4, "little") for v in (logD, Q, R)))
    return [T.challenges(t, logD) for t in ("relu/uZ", "relu/uA", "relu/uGA", "relu/uGZ")]


def verify_relu(tr: HostTranscript, proof: bytes, shape, points: list | None = None) -> dict:
    """zk_verify_relu for shape = (logD, Q, R); points: None (D3b draws them) or the chained form's given
    points (D25).  Returns dict(points, claims, point, finals) from the verified proof."""
    logD, Q, R = (int(v) for v in shape)
    if not (1 <= logD <= 40 and 1 <= Q <= 32 and 1 <= R <= 32 and Q + R <= 32):
        raise ValueError("bad zkReLU shape")
    m = max(0, (Q + R - 1).bit_length()) + logD
    pts = relu_points(tr, logD, Q, R) if points is None else [list(u) for u in points]
    pt = ctypes.create_string_buffer(32 * m)
    _run("zkReLU", lib().zk_verify_relu, tr.st, proof, len(proof), (ctypes.c_uint32 * 3)(logD, Q, R),
         None if points is None else _fr([x for u in points for x in u]), pt)
    claims = [int.from_bytes(proof[12 + 32 * i:44 + 32 * i], "little") for i in range(4)]
    return dict(points=pts, claims=claims, point=_ints(pt, m), finals=_fin(proof, 3))


def verify_loss_grad(tr: HostTranscript, m: int, claims: list) -> list:
    """zk_verify_loss_grad (D24): returns the point u; raises Rejected unless G_Z~(u) = Z~(u) - Y~(u)."""
    pt = ctypes.create_string_buffer(32 * m)
    _run("loss gradient", lib().zk_verify_loss_grad, tr.st, m, _fr(claims), pt)
    return _ints(pt, m)


def verify_relu_merge(tr: HostTranscript, logD: int, Q: int, R: int, relu_point: list, relu_finals: list,
                      proof: bytes) -> dict:
    """zk_verify_relu_merge (D21): returns dict(point = (r_j, r_s), claim = aux~(r_s, v, r_j), weight)."""
    m = max(0, (Q + R - 1).bit_length()) + 1
    pt = ctypes.create_string_buffer(32 * m)
    _run("zkReLU merge", lib().zk_verify_relu_merge, tr.st, logD, Q, R, _fr(relu_point), _fr(relu_finals), proof,
         len(proof), pt)
    f = _fin(proof, 2)
    return dict(point=_ints(pt, m), claim=f[0], weight=f[1])


def verify_rescale(tr: HostTranscript, proof: bytes, shape, points: list) -> dict:
    """zk_verify_rescale (D26) for shape = (logD, Q, R) at the given points (u_Z, u_P).  Returns dict(claims =
    [Z~(u_Z), Z'~(u_P)], aux = [aux~(r_A), aux~(r_B)], rA, rB) from the verified proof."""
    logD, Q, R = (int(v) for v in shape)
    if not (1 <= logD <= 40 and 1 <= Q <= 32 and 1 <= R <= 32 and Q + R <= 32):
        raise ValueError("bad rescale shape")
    m = max(0, (Q + R - 1).bit_length()) + logD
    cl, aux, pt = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64), ctypes.create_string_buffer(64 * m)
    _run("rescale", lib().zk_verify_rescale, tr.st, proof, len(proof), (ctypes.c_uint32 * 3)(logD, Q, R),
         _fr([x for u in points for x in u]), cl, aux, pt)
    p2 = _ints(pt, 2 * m)
    return dict(claims=_ints(cl, 2), aux=_ints(aux, 2), rA=p2[:m], rB=p2[m:])


def verify_claim_merge(tr: HostTranscript, n: int, d: int, claims: list, proof: bytes) -> tuple:
    """zk_verify_claim_merge (D25).  claims: dicts(map, v (d elements), u (log2 len(map)), c).
    Returns (point (d + n), claim): the one claim left on the stack."""
    from ._lib import CmView
    K = len(claims)
    arrs = [(ctypes.c_uint32 * len(c["map"]))(*[int(i) & 0xFFFFFFFF for i in c["map"]]) for c in claims]
    views = (CmView * K)(*[CmView(len(c["map"]).bit_length() - 1, ctypes.cast(a, ctypes.c_void_p))
                           for c, a in zip(claims, arrs)])
    pts = [x for c in claims for x in list(c["v"]) + list(c["u"])]
    pt, cl = ctypes.create_string_buffer(32 * (d + n)), ctypes.create_string_buffer(32)
    _run("claim merge", lib().zk_verify_claim_merge, tr.st, n, d, K, views, _fr(pts), _fr([c["c"] for c in claims]),
         proof, len(proof), pt, cl)
    return _ints(pt, d + n), _ints(cl, 1)[0]


def verify_matmul(tr: HostTranscript, logs, res: dict) -> dict:
    """A matmul family (rows a3-a6): the verifier draws w, u1, u3 itself (D3a), checks they are the
    prover's, then verifies the product sumcheck (m = logN + logD2, n_eq = logN, K = 2) of the proof's
    claim Y~(w, u1, u3).  Returns dict(w, u1, u3, claim, r, finals) — claim and finals from the proof."""
    lN, l1, l2, l3 = logs
    tr.absorb("mm/hdr", b"".join(int(v).to_bytes(4, "little") for v in (lN, l1, l2, l3)))
    w, u1, u3 = tr.challenges("mm/w", lN), tr.challenges("mm/u1", l1), tr.challenges("mm/u3", l3)
    if (w, u1, u3) != (res["w"], res["u1"], res["u3"]):
        raise Rejected("matmul points", -2)
    proof = res["proof"]
    r = verify_sumcheck(tr, proof, w, shape=(lN + l2, lN, 2))
    return dict(w=w, u1=u1, u3=u3, claim=int.from_bytes(proof[12:44], "little"), r=r, finals=_fin(proof, 2))


def _family_logs(f):
    from .api import _mm_logs
    ta, tb = getattr(f, "trans_a", getattr(f, "transA", False)), getattr(f, "trans_b", getattr(f, "transB", False))
    return _mm_logs(f.A, f.B, ta, tb), ta, tb


def _relu_shape(f):
    return int(f.Z.size if hasattr(f.Z, "size") and not callable(f.Z.size) else f.Z.numel()).bit_length() - 1, f.Q, f.R


def verify_window(seed: bytes, header: bytes, families: list, results: list) -> list:
    """Replays a D3d window: W absorbs "fcn/hdr", per family "fcn/fam" and forks "fcn/fork"; each
    family's proof is verified on its own forked transcript and must end in the state the prover
    reported; W absorbs "fcn/join" of every family and must end in the reported window state.
    families: the window's family records (shapes only are read); results: fcn.prove_window's output.
    Returns per family every claim it leaves open (the D3d window binds no claim to another family's):
    matmul: the claim Y~(w, u1, u3) with (w, u1, u3), the point r and the finals A~, B~ there; ReLU: the
    four claims with their points, the final point and the aux finals (+ the aux merge)."""
    W = HostTranscript(seed=seed)
    W.absorb("fcn/hdr", header)
    kids = []
    for f in families:
        W.absorb("fcn/fam", f.name.encode())
        kids.append(W.fork("fcn/fork"))
    out = []
    for f, T, res in zip(families, kids, results):
        if hasattr(f, "A"):   # a matmul family (device record or host synth.fcn record: shapes only)
            logs, _, _ = _family_logs(f)
            v = verify_matmul(T, logs, res)
            out.append(dict(name=f.name, w=v["w"], u1=v["u1"], u3=v["u3"], claim=v["claim"], point=v["r"],
                            finals=v["finals"]))
        else:
            shape = _relu_shape(f)
            v = verify_relu(T, res["proof"], shape)
            item = dict(name=f.name, points=v["points"], claims=v["claims"], point=v["point"], finals=v["finals"])
            if "merge" in res:
                mg = verify_relu_merge(T, shape[0], f.Q, f.R, v["point"], v["finals"], res["merge"]["proof"])
                item["merge_point"], item["merge_claim"] = mg["point"], mg["claim"]
            out.append(item)
        if T.state() != res["state"]:
            raise Rejected(f"family {f.name} transcript state", -3)
    for T in kids:
        W.absorb("fcn/join", T.state())
    if W.state() != results[-1]["window_state"]:
        raise Rejected("window transcript state", -3)
    return out


def verify_window_chained(seed: bytes, header: bytes, families: list, tensors: list, res: dict) -> dict:
    """Replays a claim-chained window (Protocol 1 lines 7-8, D25; chain.prove_window_chained's
    output `res`).  families: records with shapes and refs (synth.fcn after plan_window, or
    chain.ChainedFamily); tensors: the plan's tensor families (name, slots/pad, rows, cols, relu).
    Every matmul family is verified on its fork; the claims it leaves are routed by the plan to their
    tensor families; every tensor family with more than one claim (or one on a partial view) must carry a
    verified claim merge of exactly those claims; every ReLU family is verified at the merged points of
    its Z, A, G_A, G_Z stacks and its four claims must EQUAL the merged claims (nothing unbound); its aux
    merge gives the aux claim.  Returns {tensor family: (point, value)} for every committed stack and
    {"aux:<ReLU>": (point over (j, i, s), value)} — exactly the claims left for the commitments."""
    from .plan import RELU_ROLES, family_kind, is_whole, matmul_claim_pieces
    W = HostTranscript(seed=seed)
    W.absorb("fcn/chdr", header)
    mms = [f for f in families if family_kind(f) == "matmul"]
    losses = [f for f in families if family_kind(f) == "loss"]
    relus = [f for f in families if family_kind(f) == "relu"]
    rescales = [f for f in families if family_kind(f) == "rescale"]

    def refs(f):
        return {k: (v.tensor, list(v.map)) if hasattr(v, "tensor") else (v[0], list(v[1])) for k, v in f.refs.items()}

    def pad_of(t):
        return list(t.pad) if hasattr(t, "pad") else [s is None for s in t.slots]

    kids = []
    for f in mms + losses:
        W.absorb("fcn/fam", f.name.encode())
        kids.append(W.fork("fcn/fork"))
    claims = {t.name: [] for t in tensors}
    for f, T in zip(mms, kids):
        r = res["matmul"][f.name]
        logs, ta, tb = _family_logs(f)
        v = verify_matmul(T, logs, r)
        if T.state() != r["state"]:
            raise Rejected(f"family {f.name} transcript state", -3)
        lN = logs[0]
        val = dict(w=v["w"], u1=v["u1"], u3=v["u3"], claim=[v["claim"]], fA=[v["finals"][0]], fB=[v["finals"][1]],
                   rn=v["r"][:lN], rk=v["r"][lN:])
        rf = refs(f)
        for role, vp, up, cp in matmul_claim_pieces(ta, tb):
            tname, mp = rf[role]
            claims[tname].append(dict(map=mp, v=[x for p in vp for x in val[p]], u=[x for p in up for x in val[p]],
                                      c=val[cp][0]))
    for f, T in zip(losses, kids[len(mms):]):
        r = res["loss"][f.name]
        n = int(f.GZ.size if not callable(f.GZ.size) else f.GZ.numel())
        d = int(f.GZ.shape[1] * f.GZ.shape[2]).bit_length() - 1
        u = verify_loss_grad(T, n.bit_length() - 1, r["claims"])
        if T.state() != r["state"]:
            raise Rejected(f"family {f.name} transcript state", -3)
        rf = refs(f)
        for role, c in zip(("GZ", "Zp", "Y"), r["claims"]):
            tname, mp = rf[role]
            claims[tname].append(dict(map=mp, v=u[:d], u=u[d:], c=c))
    for T in kids:
        W.absorb("fcn/join", T.state())
    opened = {}
    merged = []
    for t in tensors:
        cl = claims[t.name]
        if not cl:
            continue
        if is_whole(pad_of(t), [c["map"] for c in cl]):
            opened[t.name] = (cl[0]["v"] + cl[0]["u"], cl[0]["c"])
        else:
            merged.append(t)
    if set(res["merges"]) != {t.name for t in merged}:
        raise Rejected("claim merges do not match the window plan", -4)
    # D25 order: the merges stage 3 is bound to, joined before stage 3; the other merges forked after stage
    # 3's families (they prove beside it) and joined after them
    bound = {f.tensors[k] for f in relus for k in RELU_ROLES} | {f.tensors[k] for f in rescales for k in ("Z", "Zp")}
    merged_a = [t for t in merged if t.name in bound]
    merged_b = [t for t in merged if t.name not in bound]

    def check_merges(ts, ks):
        for t, T in zip(ts, ks):
            n = len(pad_of(t)).bit_length() - 1
            d = (t.rows * t.cols).bit_length() - 1
            mr = res["merges"][t.name]
            opened[t.name] = verify_claim_merge(T, n, d, claims[t.name], mr["proof"])
            if T.state() != mr["state"]:
                raise Rejected(f"claim merge {t.name} transcript state", -3)

    kids2 = []
    for t in merged_a:
        W.absorb("fcn/tfam", t.name.encode())
        kids2.append(W.fork("fcn/fork"))
    check_merges(merged_a, kids2)
    for T in kids2:
        W.absorb("fcn/join", T.state())
    kids3 = []
    for f in relus + rescales:
        W.absorb("fcn/fam", f.name.encode())
        kids3.append(W.fork("fcn/fork"))
    kids2b = []
    for t in merged_b:
        W.absorb("fcn/tfam", t.name.encode())
        kids2b.append(W.fork("fcn/fork"))
    check_merges(merged_b, kids2b)
    for f, T in zip(rescales, kids3[len(relus):]):
        r = res["rescale"][f.name]
        names = [f.tensors["Z"], f.tensors["Zp"]]
        if any(nm not in opened for nm in names):
            raise Rejected(f"{f.name}: a rescale-bound stack without a claim", -4)
        n = int(f.Z.size if not callable(f.Z.size) else f.Z.numel())
        logB = max(0, (f.Q + f.R - 1).bit_length())
        v = verify_rescale(T, r["proof"], (n.bit_length() - 1, f.Q, f.R), [opened[nm][0] for nm in names])
        if v["claims"] != [opened[nm][1] for nm in names]:
            raise Rejected(f"{f.name}: rescale claims differ from the window's claims", -1)
        aux = [dict(map=[0], u=[], v=v["rA"], c=v["aux"][0]), dict(map=[0], u=[], v=v["rB"], c=v["aux"][1])]
        pt, cl = verify_claim_merge(T, 0, (n.bit_length() - 1) + logB, aux, r["aux_merge"]["proof"])
        if T.state() != r["state"]:
            raise Rejected(f"family {f.name} transcript state", -3)
        for nm in names:
            del opened[nm]
        opened["aux:" + f.name] = (pt, cl)
    for f, T in zip(relus, kids3):
        r = res["relu"][f.name]
        names = [f.tensors[k] for k in RELU_ROLES]
        if any(nm not in opened for nm in names):
            raise Rejected(f"{f.name}: a ReLU-bound stack without a claim", -4)
        shape = _relu_shape(f)
        v = verify_relu(T, r["proof"], shape, points=[opened[nm][0] for nm in names])
        if v["claims"] != [opened[nm][1] for nm in names]:
            raise Rejected(f"{f.name}: zkReLU claims differ from the merged claims", -1)
        mg = verify_relu_merge(T, shape[0], f.Q, f.R, v["point"], v["finals"], r["merge"]["proof"])
        if T.state() != r["state"]:
            raise Rejected(f"family {f.name} transcript state", -3)
        for nm in names:            # bound through zkReLU by the aux commitment: not opened
            del opened[nm]
        logB = max(0, (f.Q + f.R - 1).bit_length())
        opened["aux:" + f.name] = (mg["point"][:logB] + v["point"][logB:] + mg["point"][logB:], mg["claim"])
    for T in kids3 + kids2b:
        W.absorb("fcn/join", T.state())
    if W.state() != res["window_state"]:
        raise Rejected("window transcript state", -3)
    return opened
