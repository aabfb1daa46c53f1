"""Oracle drivers for the named configurations — TEST INFRASTRUCTURE ONLY.

They string the oracle's per-protocol calls together in the order DESIGN.md
fixes (D3a matmul, D3b zkReLU, D3c single sumcheck, D3d FCN families), on
inputs from synth/ (the shared seeded generators).
"""
from __future__ import annotations

import numpy as np

import oracle as O
from synth.fcn import LossFamily, MatmulFamily, ReluFamily, RescaleFamily, fcn_header
from synth.prng import DATA_SEED, fs_seed, uniform_range

P = O.P


def c1_inputs(seed=DATA_SEED):
    """C1: A [32][64] @ B [64][64], 16-bit entries, N = 1 (BASELINE.json configs[0])."""
    A = uniform_range(seed, 1, (1, 32, 64), -(1 << 15), 1 << 15)
    B = uniform_range(seed, 2, (1, 64, 64), -(1 << 15), 1 << 15)
    return A, B


def c2_inputs(seed=DATA_SEED, D=64 * 1024):
    """C2: one zkReLU layer, batch 64 x width 1024, Z and G_A over all 32 bit-columns."""
    Z = uniform_range(seed, 11, (D,), -(1 << 31), 1 << 31)
    GA = uniform_range(seed, 12, (D,), -(1 << 31), 1 << 31)
    return Z, GA


def c5_inputs(m: int, seed=DATA_SEED):
    """C5: A, B [2^m] int32 ~ U[-2^15, 2^15)."""
    A = uniform_range(seed, 21, (1 << m,), -(1 << 15), 1 << 15)
    B = uniform_range(seed, 22, (1 << m,), -(1 << 15), 1 << 15)
    return A, B


def embed_i32_bytes(v: np.ndarray) -> bytes:
    """Canonical 32-byte LE encodings of int32 values (negatives -> p - |v|), vectorised."""
    v = np.asarray(v, dtype=np.int64).reshape(-1)
    limbs = np.zeros((v.size, 4), dtype=np.uint64)
    pl = [(P >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(4)]
    neg = v < 0
    limbs[:, 0] = np.where(neg, np.uint64(pl[0]) - np.abs(v).astype(np.uint64), v.astype(np.uint64))
    for i in range(1, 4):
        limbs[:, i] = np.where(neg, np.uint64(pl[i]), np.uint64(0))
    return limbs.astype("<u8").tobytes()


def c1_prove(seed_name="C1"):
    A, B = c1_inputs()
    tr = O.Transcript(fs_seed(seed_name))
    res = O.matmul_prove(tr, A, B)
    res["state"] = tr.state()
    return res


def c2_prove(D=64 * 1024, seed_name="C2"):
    Z, GA = c2_inputs(D=D)
    tr = O.Transcript(fs_seed(seed_name))
    res = O.relu_prove(tr, Z, GA, 16, 16)
    res["state"] = tr.state()
    return res


def single_sumcheck_i32(tr: O.Transcript, A: np.ndarray, B: np.ndarray, tag_prefix="c5"):
    """D3c: "<p>/hdr" (m) | w = "<p>/w" x m | product sumcheck n_eq = m, K = 2, claim computed."""
    m = A.size.bit_length() - 1
    tr.absorb(f"{tag_prefix}/hdr", int(m).to_bytes(4, "little"))
    w = tr.challenges(f"{tag_prefix}/w", m)
    ta = O.from_bytes(embed_i32_bytes(A))
    tb = O.from_bytes(embed_i32_bytes(B))
    res = O.sumcheck_prove(tr, m, m, [ta, tb], w, None)
    res["w"] = w
    return res


def c5_prove(m: int):
    A, B = c5_inputs(m)
    tr = O.Transcript(fs_seed(f"C5-m{m}"))
    res = single_sumcheck_i32(tr, A, B)
    res["state"] = tr.state()
    return res


def fcn_prove(shape, families, seed_name: str, only=None, merge_aux: bool = False):
    """D3d: window transcript W: "fcn/hdr"; per family (in order) "fcn/fam" <name> and a fork: the family
    transcript T_f is seeded with the canonical bytes of W's challenge "fcn/fork"; each family's protocol
    runs on its own T_f; finally W absorbs "fcn/join" <T_f state> for every family (in order).
    Returns the per-family results (res["state"] = T_f's final state) and, as the last entry's
    "window_state", W's final state."""
    W = O.Transcript(fs_seed(seed_name))
    W.absorb("fcn/hdr", fcn_header(shape))
    fams = list(families if only is None else families[:only])
    forks = []
    for f in fams:
        W.absorb("fcn/fam", f.name.encode())
        c = W.challenges("fcn/fork", 1)[0]
        forks.append(O.Transcript(c.to_bytes(32, "little")))
    out = []
    for f, T in zip(fams, forks):
        if isinstance(f, MatmulFamily):
            res = O.matmul_prove(T, f.A, f.B, f.transA, f.transB)
        else:
            res = O.relu_prove(T, f.Z, f.GA, f.Q, f.R)
            if merge_aux:   # DESIGN.md D21: the aux-claim merge on the family transcript
                res["merge"] = O.relu_merge(T, f.Z, f.GA, f.Q, f.R, res["point"], res["finals"])
        res["name"] = f.name
        res["state"] = T.state()
        out.append(res)
    for T in forks:
        W.absorb("fcn/join", T.state())
    if out:
        out[-1]["window_state"] = W.state()
    return out


# ---------------------------------------------------------------- N3: the claim-chained window (D25)
def _matmul_family_claims(f, res):
    """The three claims a matmul family's proof leaves (Eq. exm-matmul-batched): Y~(w, u1, u3) (the
    claim it started from) and the operand finals A~(r_n, u1, r_k), B~(r_n, r_k, u3), each as a claim on a
    view of a tensor family: (role, ref, inner point over the stored [rows][cols] slice (col bits, row
    bits, D2), slot point, value)."""
    lN = res["logs"][0]
    rn, rk = res["r"][:lN], res["r"][lN:]
    vA = res["u1"] + rk if f.transA else rk + res["u1"]
    vB = rk + res["u3"] if f.transB else res["u3"] + rk
    return [("Y", f.refs["Y"], res["u3"] + res["u1"], res["w"], res["claim"]),
            ("A", f.refs["A"], vA, rn, res["finals"][0]),
            ("B", f.refs["B"], vB, rn, res["finals"][1])]


def _is_whole(t, cl):
    """One claim whose view is the whole stack (slot j -> j; an empty slot only where the stack pads)."""
    if len(cl) != 1 or len(cl[0]["map"]) != len(t.slots):
        return False
    return all((i == j) if i >= 0 else t.slots[j] is None for j, i in enumerate(cl[0]["map"]))


def _tensor_values(t, families):
    """The int32 stack [N][rows * cols] of a tensor family; the ReLU-bound ones from the words (Lemma 1),
    the rescaled top output Z' from the rescale family's Z (D9)."""
    N = len(t.slots)
    if t.array is not None:
        return np.ascontiguousarray(t.array.reshape(N, -1))
    f = next(g for g in families if g.name == t.relu)
    if t.kind == "Zp":
        z = np.asarray(f.Z, dtype=np.int64)
        return np.ascontiguousarray(((z + (1 << (f.R - 1))) >> f.R).astype(np.int32).reshape(N, -1))
    if t.kind in ("Z", "GA"):
        v = f.Z if t.kind == "Z" else f.GA
    else:
        tb = O.relu_tables(f.Z, f.GA, f.Q, f.R)
        v = tb["A"] if t.kind == "A" else tb["GZ"]
    return np.ascontiguousarray(np.asarray(v, dtype=np.int32).reshape(N, -1))


def _loss_family_claims(f, res):
    """The loss family's three claims (D24) at its point u = (inner bits, slot bits) of the stacked
    [N][B][d_L] tensors."""
    d = (f.GZ.shape[1] * f.GZ.shape[2]).bit_length() - 1
    u = res["u"]
    return [(role, f.refs[role], u[:d], u[d:], c) for role, c in zip(("GZ", "Zp", "Y"), res["claims"])]


def fcn_prove_chained(shape, families, tensors, seed_name: str, top=None):
    """The claim-chained window (Protocol 1 lines 7-8; D25).  Window transcript W:
    "fcn/chdr" (header) | stage 1: per matmul family "fcn/fam" <name> and a fork; each family proved on
    its fork (D3a) | "fcn/join" per family | stage 2: per tensor family whose claims need merging (more
    than one claim, or one claim on a view that is not the whole stack) AND that stage 3 is bound to (a ReLU
    family's Z, A, G_A, G_Z, the rescale's Z, Z') "fcn/tfam" <name> and a fork; the claim merge (D25) on it
    | joins | stage 3: per ReLU family "fcn/fam" <name> and a fork; the chained zkReLU (points = the merged
    claims of its Z, A, G_A, G_Z stacks) and the aux merge (D21) on it; the rescale likewise; then
    "fcn/tfam" <name> and a fork per remaining merge (the other tensor families, independent of stage 3) |
    joins of stage 3, then of those merges.  Returns dict(matmul, merges, relu (per family name), opened: tensor family -> (point, value)
    for every committed stack and "aux:<ReLU family>" (one claim per tensor family, Protocol 1 line 10),
    window_state)."""
    W = O.Transcript(fs_seed(seed_name))
    W.absorb("fcn/chdr", fcn_header(shape))
    top = list(top or [])
    mms = [f for f in families if isinstance(f, MatmulFamily)]
    relus = [f for f in families if isinstance(f, ReluFamily)]
    losses = [f for f in top if isinstance(f, LossFamily)]
    rescales = [f for f in top if isinstance(f, RescaleFamily)]

    def fork():
        return O.Transcript(W.challenges("fcn/fork", 1)[0].to_bytes(32, "little"))

    kids = []
    for f in mms + losses:
        W.absorb("fcn/fam", f.name.encode())
        kids.append(fork())
    mres = {}
    for f, T in zip(mms + losses, kids):
        if isinstance(f, LossFamily):
            r = O.loss_grad_prove(T, f.GZ, f.Zp, f.Y)
        else:
            r = O.matmul_prove(T, f.A, f.B, f.transA, f.transB)
        r["state"] = T.state()
        mres[f.name] = r
    for T in kids:
        W.absorb("fcn/join", T.state())
    claims = {t.name: [] for t in tensors}
    for f in mms + losses:
        fc = _loss_family_claims(f, mres[f.name]) if isinstance(f, LossFamily) else _matmul_family_claims(f, mres[f.name])
        for role, ref, v, u, c in fc:
            claims[ref.tensor].append(dict(map=list(ref.map), u=list(u), v=list(v), c=c, src=(f.name, role)))
    opened = {}
    to_merge = []
    for t in tensors:
        cl = claims[t.name]
        if not cl:
            continue
        if _is_whole(t, cl):
            opened[t.name] = (cl[0]["v"] + cl[0]["u"], cl[0]["c"])
        else:
            to_merge.append(t)
    # stage 2 splits (D25, round-2 order): the merges of the stacks stage 3 is bound to (the ReLU families'
    # Z, A, G_A, G_Z and the rescale's Z, Z') come first and are joined; the other merges are forked after
    # stage 3's families, so they prove beside it
    bound = {f.tensors[k] for f in relus for k in ("Z", "A", "GA", "GZ")} | \
        {f.tensors[k] for f in rescales for k in ("Z", "Zp")}
    merge_a = [t for t in to_merge if t.name in bound]
    merge_b = [t for t in to_merge if t.name not in bound]
    merges = {}

    def prove_merges(ts, ks):
        for t, T in zip(ts, ks):
            r = O.claim_merge_prove(T, _tensor_values(t, families), claims[t.name])
            r["state"] = T.state()
            r["claims_in"] = claims[t.name]
            merges[t.name] = r
            opened[t.name] = (r["point"], r["claim"])

    mk = []
    for t in merge_a:
        W.absorb("fcn/tfam", t.name.encode())
        mk.append(fork())
    prove_merges(merge_a, mk)
    for T in mk:
        W.absorb("fcn/join", T.state())
    rk = []
    for f in relus + rescales:
        W.absorb("fcn/fam", f.name.encode())
        rk.append(fork())
    mkb = []
    for t in merge_b:
        W.absorb("fcn/tfam", t.name.encode())
        mkb.append(fork())
    prove_merges(merge_b, mkb)
    rres = {}
    for f, T in zip(relus + rescales, rk):
        if isinstance(f, RescaleFamily):   # D26, then the claim merge (D25) of its two aux claims
            names = [f.tensors["Z"], f.tensors["Zp"]]
            r = O.rescale_prove(T, f.Z, f.Q, f.R, [opened[n][0] for n in names])
            logB = O.relu_logB(f.Q, f.R)
            D = f.Z.size
            bits = ((f.Z.astype(np.int64).reshape(-1, 1) & 0xFFFFFFFF) >> np.arange(1 << logB)) & 1
            bits[:, f.Q + f.R:] = 0
            aux = [dict(map=[0], u=[], v=r["A"]["r"], c=r["A"]["finals"][1]),
                   dict(map=[0], u=[], v=r["B"]["r"], c=r["B"]["finals"][0])]
            r["aux_merge"] = O.claim_merge_prove(T, np.ascontiguousarray(bits.astype(np.int32).reshape(1, D << logB)), aux)
            r["state"] = T.state()
            rres[f.name] = r
            for n in names:
                opened.pop(n)
            opened["aux:" + f.name] = (r["aux_merge"]["point"], r["aux_merge"]["claim"])
            continue
        names = [f.tensors[k] for k in ("Z", "A", "GA", "GZ")]
        r = O.relu_prove(T, f.Z, f.GA, f.Q, f.R, points=[opened[n][0] for n in names])
        r["merge"] = O.relu_merge(T, f.Z, f.GA, f.Q, f.R, r["point"], r["finals"])
        r["state"] = T.state()
        rres[f.name] = r
        for n in names:          # bound by the aux commitment through zkReLU: not opened
            opened.pop(n)
        logB = O.relu_logB(f.Q, f.R)
        rj, rs = r["merge"]["r"][:logB], r["merge"]["r"][logB:]
        opened["aux:" + f.name] = (rj + r["point"][logB:] + rs, r["merge"]["finals"][0])
    for T in rk + mkb:
        W.absorb("fcn/join", T.state())
    return dict(matmul=mres, merges=merges, relu=rres, opened=opened, window_state=W.state())
