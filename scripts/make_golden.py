"""Write tests/golden/*.json from the ORACLE ONLY (never from the CUDA path).

    python scripts/make_golden.py

c1_transcript.json: the full C1 proof (single matmul sumcheck 32x64 @ 64x64,
16-bit entries, FS seed SHA256("zkdl-b200/fs-seed/C1")) — BASELINE.json configs[0].
relu_small.json:    a zkReLU proof at D = 2^6, Q = R = 16 (C2's statement at a tiny size).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from oracle import drivers  # noqa: E402
from synth.prng import fs_seed  # noqa: E402


def main():
    out = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out, exist_ok=True)
    res = drivers.c1_prove()
    doc = {
        "source": "scripts/make_golden.py -> oracle/ (oracle.c); DESIGN.md D2-D4, D3a",
        "config": "C1: single matmul sumcheck 32x64 @ 64x64, 16-bit entries, N=1",
        "fs_seed": fs_seed("C1").hex(),
        "w": [hex(v) for v in res["w"]], "u1": [hex(v) for v in res["u1"]], "u3": [hex(v) for v in res["u3"]],
        "claim": hex(res["claim"]),
        "msgs": [[hex(v) for v in row] for row in res["msgs"]],
        "r": [hex(v) for v in res["r"]],
        "finals": [hex(v) for v in res["finals"]],
        "final_state": res["state"].hex(),
    }
    with open(os.path.join(out, "c1_transcript.json"), "w") as f:
        json.dump(doc, f, indent=1)
    r2 = drivers.c2_prove(D=64, seed_name="C2-small")
    doc2 = {
        "source": "scripts/make_golden.py -> oracle/ (oracle.c); DESIGN.md D3b, D5, D10, D12, D13",
        "config": "zkReLU D=64, Q=R=16, inputs = C2 generator truncated to 64 entries",
        "claims": [hex(v) for v in r2["claims"]],
        "msgs": [[hex(v) for v in row] for row in r2["msgs"]],
        "point": [hex(v) for v in r2["point"]],
        "finals": [hex(v) for v in r2["finals"]],
        "final_state": r2["state"].hex(),
    }
    with open(os.path.join(out, "relu_small.json"), "w") as f:
        json.dump(doc2, f, indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
