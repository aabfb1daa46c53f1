"""Claim bookkeeping of the claim-chained window (D25) shared by the device
driver (chain.py) and the host verifier (verify.py).  Structure only: which proof output is which claim.

A matmul family's proof (Eq. exm-matmul-batched; transcript D3a) leaves three claims, each on a
view of a tensor family (synth.fcn.plan_window's refs), named by the pieces of the family's output:
    Y:  Y~(w, u1, u3)   inner point (u3, u1) over the stored [D1][D3] slice, slot point w, value "claim"
    A:  A~(r_n, u1, r_k) inner (r_k, u1) over [D1][D2] ((u1, r_k) when A is stored transposed), "fA"
    B:  B~(r_n, r_k, u3) inner (u3, r_k) over [D2][D3] ((r_k, u3) when B is stored transposed), "fB"
with r = (r_n, r_k) the product sumcheck's point (the stack variables are bound first, Protocol 2-3) and
every inner point ordered (col bits, row bits) of the slice as stored (D2).
"""
from __future__ import annotations


def matmul_claim_pieces(trans_a: bool, trans_b: bool) -> list:
    """[(role, inner point pieces, slot point pieces, value piece)] in the fixed order Y, A, B."""
    return [("Y", ["u3", "u1"], ["w"], "claim"),
            ("A", ["u1", "rk"] if trans_a else ["rk", "u1"], ["rn"], "fA"),
            ("B", ["rk", "u3"] if trans_b else ["u3", "rk"], ["rn"], "fB")]


def is_whole(pad: list, maps: list) -> bool:
    """True when the only claim on a tensor family is on the whole stack (slot j -> j; an empty slot only
    where the stack itself is zero padding): that claim needs no merge."""
    if len(maps) != 1 or len(maps[0]) != len(pad):
        return False
    return all((i == j) if i >= 0 else pad[j] for j, i in enumerate(maps[0]))


RELU_ROLES = ("Z", "A", "GA", "GZ")   # the order of zkReLU's points u_Z, u_A, u_GA, u_GZ (D3b)


def family_kind(f) -> str:
    """"matmul", "relu", "loss" or "rescale" for a synth.fcn family record or a device record."""
    k = getattr(f, "kind", None)
    if k:
        return k
    if getattr(f, "A", None) is not None:
        return "matmul"
    if getattr(f, "Zp", None) is not None and getattr(f, "GZ", None) is not None:
        return "loss"
    return "relu" if getattr(f, "GA", None) is not None else "rescale"
