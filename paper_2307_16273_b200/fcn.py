"""FAC4DNN family driver (PAPER Example 2 P:L292-312, Protocol 1 line 7 P:L326).

One Fiat-Shamir transcript per proving window (D3d): "fcn/hdr", then for every
family in the fixed order of synth.fcn.assemble_families, "fcn/fam" <name>
followed by the family's protocol — matmul families: zk_matmul_reduce then
zk_sumcheck_prove (m = logN + logD2, n_eq = logN, K = 2); ReLU families:
zk_relu_prove.  Stack tensors must already be resident on the device; this
module only sequences the library calls (no arithmetic here).
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
    """Copy synth.fcn families (numpy int32 stacks) to the device."""
    out = []

    def dev(a):
        t = torch.from_numpy(a)
        if pin:
            t = t.pin_memory()
        return t.to(device, non_blocking=pin)

    for f in families:
        if hasattr(f, "A"):
            out.append(DeviceFamily(f.name, "matmul", A=dev(f.A), B=dev(f.B), trans_a=f.transA, trans_b=f.transB))
        else:
            out.append(DeviceFamily(f.name, "relu", Z=dev(f.Z), GA=dev(f.GA), Q=f.Q, R=f.R))
    return out


def prove_window(ctx: api.Context, seed: bytes, header: bytes, families: list, keep_tables: bool = False) -> list:
    """Prove every family of one window under one transcript; returns per-family results."""
    tr = api.Transcript(ctx, seed)
    tr.absorb("fcn/hdr", header)
    results = []
    for f in families:
        tr.absorb("fcn/fam", f.name.encode())
        if f.kind == "matmul":
            red = api.matmul_reduce(ctx, tr, f.A, f.B, f.trans_a, f.trans_b)
            lN, _, l2, _ = red["logs"]
            sc = api.sumcheck_prove(ctx, tr, lN + l2, lN, [red["At"], red["Bt"]], red["w"], red["claim"])
            res = dict(name=f.name, kind="matmul", w=red["w"], u1=red["u1"], u3=red["u3"], claim=red["claim"],
                       msgs=sc["msgs"], r=sc["r"], finals=sc["finals"], proof=sc["proof"])
            if keep_tables:
                res["At"], res["Bt"] = red["At"], red["Bt"]
        else:
            rr = api.relu_prove(ctx, tr, f.Z, f.GA, f.Q, f.R)
            res = dict(name=f.name, kind="relu", claims=rr["claims"], msgs=rr["msgs"], point=rr["point"],
                       finals=rr["finals"], proof=rr["proof"])
        res["state"] = tr.state()
        results.append(res)
    tr.close()
    return results
