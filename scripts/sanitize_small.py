"""Small invocations of the persistent (spin-waiting) kernels for compute-sanitizer runs
(VERDICT r1 item 10): k_sc_all (product sumcheck <= 2^18 entries), k_relu_ipersist / k_relu_itail
(zkReLU i-rounds <= 2^16 pairs), each checked against the oracle so a sanitizer-perturbed schedule
that changed a result would also show."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
from oracle import drivers  # noqa: E402
from paper_2307_16273_b200 import api  # noqa: E402
from synth.prng import fs_seed, uniform_range  # noqa: E402

ctx = api.Context(0)
m = int(os.environ.get("SAN_M", "12"))
A, B = drivers.c5_inputs(m)
tr = api.Transcript(ctx, fs_seed(f"C5-m{m}"))
tr.absorb("c5/hdr", m.to_bytes(4, "little"))
w = tr.challenges("c5/w", m)
g = api.sumcheck_prove(ctx, tr, m, m, [torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()], w)
o = drivers.c5_prove(m)
assert g["msgs"] == o["msgs"] and g["finals"] == o["finals"], "k_sc_all parity"
logD = int(os.environ.get("SAN_LOGD", "12"))
Z = uniform_range(5, 1, (1 << logD,), -(1 << 31), 1 << 31)
GA = uniform_range(5, 2, (1 << logD,), -(1 << 31), 1 << 31)
gr = api.relu_prove(ctx, api.Transcript(ctx, fs_seed("san")), torch.from_numpy(Z).cuda(), torch.from_numpy(GA).cuda(), 16, 16)
orr = oracle.relu_prove(oracle.Transcript(fs_seed("san")), Z, GA, 16, 16)
assert gr["msgs"] == orr["msgs"] and gr["finals"] == orr["finals"], "zkReLU parity"
torch.cuda.synchronize()
print("sanitize_small ok", m, logD, ctx.launches)
