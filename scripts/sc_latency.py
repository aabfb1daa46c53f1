"""Per-round latency of the persistent small-statement sumcheck (k_sc_all) and of transcript steps, under
gpurun with ZKDL_SCALL_TRACE=1: python scripts/sc_latency.py [--m 10 14 18] [--budget 37]"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16273_b200 import api, build  # noqa: E402
from synth.prng import fs_seed, uniform_range  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, nargs="*", default=[10, 14, 18])
    ap.add_argument("--budget", type=int, default=37)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    build.build(verbose=False)
    stream = torch.cuda.Stream()
    ctx = api.Context(0, stream)
    if args.budget:
        ctx.set_sm_budget(args.budget)
    with torch.cuda.stream(stream):
        for m in args.m:
            A = torch.from_numpy(uniform_range(230716273, 21, (1 << m,), -(1 << 15), 1 << 15)).cuda()
            B = torch.from_numpy(uniform_range(230716273, 22, (1 << m,), -(1 << 15), 1 << 15)).cuda()
            for rep in range(args.reps):
                tr = api.Transcript(ctx, fs_seed(f"lat-{m}"))
                w = tr.challenges("c5/w", m)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                api.sumcheck_prove(ctx, tr, m, m, [A, B], w)
                torch.cuda.synchronize()
                print(f"m={m} rep={rep} total {1e3 * (time.perf_counter() - t0):.3f} ms "
                      f"({1e6 * (time.perf_counter() - t0) / m:.1f} us/round)", file=sys.stderr)
                tr.close()
        # transcript alone: challenges
        tr = api.Transcript(ctx, fs_seed("lat-tr"))
        for n in (1, 16):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(10):
                tr.challenges("x/y", n)
            torch.cuda.synchronize()
            print(f"challenges({n}) x10: {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr)


if __name__ == "__main__":
    main()
