"""Where the C4 window's time goes: the window (bench configuration) against the zkReLU family alone
and the matmul families alone, each timed with CUDA events over 5 windows after 3 warm-up windows.

    python scripts/window_split.py [--mm-budget 37] [--mm-streams 2]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16273_b200 import api                # noqa: E402
from paper_2307_16273_b200 import fcn as dfcn        # noqa: E402
from synth import fcn                                # noqa: E402
from synth.prng import DATA_SEED, fs_seed            # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mm-budget", type=int, nargs="+", default=[37])
ap.add_argument("--mm-streams", type=int, nargs="+", default=[2])
args = ap.parse_args()
shape = fcn.C4_SHAPE
fams = fcn.assemble_families(shape, fcn.generate_trace(shape, seed=DATA_SEED))
dev = dfcn.upload_families(fams)
header, seed = fcn.fcn_header(shape), fs_seed("split")
ctx = api.Context(0)


def timed(fn, n=5, w=3):
    """windows enqueued back to back (as bench.py does), one synchronisation at the end"""
    keep = [fn() for _ in range(w)]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream)
    keep = [fn() for _ in range(n)]
    b.record(ctx.stream)
    torch.cuda.synchronize()
    del keep
    return a.elapsed_time(b) / n


relu = [f for f in dev if f.kind == "relu"]
mm = [f for f in dev if f.kind == "matmul"]
print(f"relu alone (full GPU): {timed(lambda: dfcn.enqueue_window(ctx, seed, header, relu)):.3f} ms")
for ns in args.mm_streams:
    for bud in args.mm_budget:
        mmc = [api.Context(0, torch.cuda.Stream()) for _ in range(ns - 1)]
        for c in [ctx] + mmc:
            c.set_sm_budget(bud)
        rc = api.Context(0, torch.cuda.Stream(priority=-1))
        t_mm = timed(lambda: dfcn.enqueue_window(ctx, seed, header, mm, mm_ctxs=mmc))
        t_all = timed(lambda: dfcn.enqueue_window(ctx, seed, header, dev, relu_ctx=rc, mm_ctxs=mmc))
        print(f"mm streams {ns} budget {bud}: matmul alone {t_mm:.3f} ms, window {t_all:.3f} ms")
        ctx.set_sm_budget(0)
