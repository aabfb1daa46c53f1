"""Kernel-level experiment bench (run under gpurun): the C4-sized zkReLU proof (D = 2^23) and a
C5 single sumcheck, with per-kernel CUDA-event times and a digest of the proof bytes, so a kernel
change can be timed and checked for identical transcripts in one call.

    python scripts/kbench.py [--logD 23] [--m 22 24] [--reps 3]
"""
import argparse
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16273_b200 import api, build  # noqa: E402
from synth.prng import fs_seed, uniform_range  # noqa: E402


def timed(ctx, fn, reps):
    ctx.profile(True)
    ctx.profile_read()
    best, out = None, None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(ctx.stream)
        out = fn()
        b.record(ctx.stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    prof = ctx.profile_read()
    ctx.profile(False)
    table = {k: round(t / reps, 4) for k, (n, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])}
    return best, out, table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--logD", type=int, default=23)
    ap.add_argument("--m", type=int, nargs="*", default=[22, 24])
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    build.build(verbose=False)
    stream = torch.cuda.Stream()
    ctx = api.Context(0, stream)
    res = {}
    with torch.cuda.stream(stream):
        if args.logD:
            D = 1 << args.logD
            Z = torch.from_numpy(uniform_range(230716273, 11, (D,), -(1 << 31), 1 << 31)).cuda()
            GA = torch.from_numpy(uniform_range(230716273, 12, (D,), -(1 << 31), 1 << 31)).cuda()
            flag = torch.zeros(1, dtype=torch.int32, device="cuda")

            def relu():
                tr = api.Transcript(ctx, fs_seed("kbench-relu"))
                out = api.relu_prove_dev(ctx, tr, Z, GA, 16, 16, flag)
                tr.close()
                return out
            relu()
            ms, out, table = timed(ctx, relu, args.reps)
            res[f"relu_logD{args.logD}"] = {"ms": round(ms, 4), "digest": hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16],
                                           "kernels_ms": table}
        for m in args.m:
            A = torch.from_numpy(uniform_range(230716273, 21, (1 << m,), -(1 << 15), 1 << 15)).cuda()
            B = torch.from_numpy(uniform_range(230716273, 22, (1 << m,), -(1 << 15), 1 << 15)).cuda()

            def c5():
                tr = api.Transcript(ctx, fs_seed(f"C5-m{m}"))
                tr.absorb("c5/hdr", m.to_bytes(4, "little"))
                w = tr.challenges("c5/w", m)
                g = api.sumcheck_prove(ctx, tr, m, m, [A, B], w)
                tr.close()
                return g
            c5()
            ms, g, table = timed(ctx, c5, args.reps)
            res[f"c5_m{m}"] = {"ms": round(ms, 4), "digest": hashlib.sha256(repr(g["msgs"]).encode()).hexdigest()[:16],
                              "kernels_ms": table}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
