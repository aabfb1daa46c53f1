"""The A/B switches of the library (environment variables read once per process) keep parity: every
alternative path a switch selects is run in a subprocess and compared with the oracle (bit-exact).

    ZKDL_SC_INT0=0       C5 round 0 through the embedding kernel instead of the integer round 0
    ZKDL_SC_DERIVE=0     product-sumcheck folding rounds with f(1) summed over the pairs (not derived from the
                         running claim)
    ZKDL_RELU_WORDS=0    zkReLU i-rounds 0/1 from materialised tables instead of the words
    ZKDL_IR_DERIVE=0     zkReLU i-rounds with every X = 1 total summed over the pairs (not derived from the
                         per-term sums)
    ZKDL_IR_CELLS=0      the first zkReLU i-round's linear terms summed over the pairs (not from the parity-split
                         bit-sum cells of the Gram kernel)
    ZKDL_MLE4_FUSED=0    the four zkReLU claims through four row-dot launches
    ZKDL_COLSUM_TC=0     column sums on the CUDA cores instead of the tensor cores (TMA + MN-major int8 MMAs)
    ZKDL_COLSUM_ROWS=0   wide CUDA-core column sums through the column-strip kernel
    ZKDL_ROWDOT_TC=0     restriction row dots on the CUDA cores instead of the tensor cores
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

C5_SNIPPET = """
import json, torch
from paper_2307_16273_b200 import api
from oracle import drivers
from synth.prng import fs_seed
m = 19
A, B = drivers.c5_inputs(m)
ctx = api.Context(0)
tr = api.Transcript(ctx, fs_seed(f"C5-m{m}"))
tr.absorb("c5/hdr", m.to_bytes(4, "little"))
w = tr.challenges("c5/w", m)
g = api.sumcheck_prove(ctx, tr, m, m, [torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()], w)
print(json.dumps({"msgs": [[str(v) for v in r] for r in g["msgs"]], "finals": [str(v) for v in g["finals"]]}))
"""

RELU_SNIPPET = """
import json, torch
from paper_2307_16273_b200 import api
from oracle import drivers
from synth.prng import fs_seed
Z, GA = drivers.c2_inputs()
ctx = api.Context(0)
g = api.relu_prove(ctx, api.Transcript(ctx, fs_seed("C2")), torch.from_numpy(Z).cuda(), torch.from_numpy(GA).cuda(), 16, 16)
print(json.dumps({"claims": [str(v) for v in g["claims"]], "msgs": [[str(v) for v in r] for r in g["msgs"]],
                  "finals": [str(v) for v in g["finals"]]}))
"""

MM_SNIPPET = """
import json, sys, torch
from paper_2307_16273_b200 import api
from synth.prng import fs_seed, uniform_range
ta, tb = bool(int(sys.argv[1])), bool(int(sys.argv[2]))
N, D1, D2, D3 = 16, 1024, 512, 1024
A = uniform_range(8, 99, (N, D2, D1) if ta else (N, D1, D2), -(1 << 15), 1 << 15)
B = uniform_range(8, 98, (N, D3, D2) if tb else (N, D2, D3), -(1 << 15), 1 << 15)
ctx = api.Context(0)
tr = api.Transcript(ctx, fs_seed("toggle-mm"))
red = api.matmul_reduce(ctx, tr, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), ta, tb)
At = api.fr_table_to_ints(ctx, red["At"]); Bt = api.fr_table_to_ints(ctx, red["Bt"])
print(json.dumps({"claim": str(red["claim"]), "At": [str(v) for v in At], "Bt": [str(v) for v in Bt]}))
"""


def run(snippet: str, env: dict, args=()) -> dict:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", snippet, *args], cwd=ROOT, env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{}, {"ZKDL_SC_INT0": "0"}, {"ZKDL_SC_DERIVE": "0"},
                                 {"ZKDL_SC_DERIVE": "0", "ZKDL_SC_INT0": "0"}])
def test_c5_paths(oracle_lib, env):
    from oracle import drivers
    o = drivers.c5_prove(19)
    g = run(C5_SNIPPET, env)
    assert g["msgs"] == [[str(v) for v in r] for r in o["msgs"]] and g["finals"] == [str(v) for v in o["finals"]]


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"ZKDL_RELU_WORDS": "0"}, {"ZKDL_MLE4_FUSED": "0"},
                                 {"ZKDL_RELU_WORDS": "0", "ZKDL_MLE4_FUSED": "0"}, {"ZKDL_IR_DERIVE": "0"},
                                 {"ZKDL_IR_DERIVE": "0", "ZKDL_RELU_WORDS": "0"}, {"ZKDL_IR_CELLS": "0"}])
def test_relu_paths(oracle_lib, env):
    from oracle import drivers
    o = drivers.c2_prove()
    g = run(RELU_SNIPPET, env)
    assert g["claims"] == [str(v) for v in o["claims"]]
    assert g["msgs"] == [[str(v) for v in r] for r in o["msgs"]] and g["finals"] == [str(v) for v in o["finals"]]


@pytest.mark.gpu
@pytest.mark.parametrize("ta,tb,env", [(0, 1, {"ZKDL_COLSUM_TC": "0", "ZKDL_COLSUM_ROWS": "0"}),
                                       (0, 1, {"ZKDL_COLSUM_TC": "0"}), (0, 1, {}),
                                       (1, 0, {"ZKDL_ROWDOT_TC": "0"}), (1, 0, {})])
def test_restriction_paths(oracle_lib, ta, tb, env):
    """The tensor-core, row-streaming and column-strip column sums (A, B^T stacks: column sums over 1024 rows
    of 512 columns), and the tensor-core and CUDA-core row dots (A^T, B stacks): the restricted tables At, Bt
    ([D2][N], every entry) and the claim equal the oracle's (or_matmul_reduce)."""
    from synth.prng import fs_seed, uniform_range
    N, D1, D2, D3 = 16, 1024, 512, 1024
    A = uniform_range(8, 99, (N, D2, D1) if ta else (N, D1, D2), -(1 << 15), 1 << 15)
    B = uniform_range(8, 98, (N, D3, D2) if tb else (N, D2, D3), -(1 << 15), 1 << 15)
    o = oracle_lib.matmul_prove(oracle_lib.Transcript(fs_seed("toggle-mm")), A, B, bool(ta), bool(tb))
    g = run(MM_SNIPPET, env, (str(ta), str(tb)))
    assert g["claim"] == str(o["claim"])
    assert g["At"] == [str(v) for v in o["At"]]
    assert g["Bt"] == [str(v) for v in o["Bt"]]
