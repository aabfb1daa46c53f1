"""Latency / throughput microbenchmarks of the Fr and transcript primitives (run under gpurun)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_16273_b200 import api, build  # noqa: E402
from paper_2307_16273_b200._lib import lib  # noqa: E402


def ev_time(fn, reps=3):
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best


def main():
    build.build(verbose=False)
    ctx = api.Context(0)
    tr = api.Transcript(ctx, bytes(32))
    out = torch.empty(32, dtype=torch.uint8, device="cuda")
    res = {}
    for mode, name in [(0, "fs_step_us"), (1, "sha256_compress_us"), (2, "fr_mul_cold_us")]:
        n = 200
        ms = ev_time(lambda: ctx.check(lib().zk_diag_fs_bench(tr.h, n, mode, out.data_ptr())))
        res[name] = 1000 * ms / n
    # register-resident Fr-mul throughput (4 chains per thread)
    import random
    P = api.P
    seed = api.fr_table_from_ints(ctx, [random.randrange(P) for _ in range(1024)])
    for blocks in (148 * 2, 148 * 4, 148 * 8):
        iters = 2000
        ms = ev_time(lambda: api.diag_mul_bench(ctx, seed, iters, blocks))
        res[f"frmul_G_per_s_blocks{blocks}"] = blocks * 256 * 4 * iters / (ms / 1000) / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
