"""Oracle drivers for the named configurations — TEST INFRASTRUCTURE ONLY.

They string the oracle's per-protocol calls together in the order DESIGN.md
fixes (D3a matmul, D3b zkReLU, D3c single sumcheck, D3d FCN families), on
inputs from synth/ (the shared seeded generators).
"""
from __future__ import annotations

import numpy as np

import oracle as O
from synth.fcn import MatmulFamily, ReluFamily, fcn_header
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
