"""The C4 window's zkReLU family alone (no matmul families beside it) against the full window: how much of
the window is the zkReLU critical path and how much the interference of the families running beside it."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2307_16273_b200 import api, build
from paper_2307_16273_b200 import fcn as dfcn
from synth import fcn
from synth.prng import fs_seed

build.build(verbose=False)
shape, fams, _ = bench.c4_workload(0)
dev = dfcn.upload_families(fams, device="cuda:0")
relu = [f for f in dev if f.kind == "relu"]
stream = torch.cuda.Stream()
ctx = api.Context(0, stream)
relu_ctx = api.Context(0, torch.cuda.Stream(priority=-1))
header = fcn.fcn_header(shape)
K = 5
for label, famset in (("zkReLU family alone", relu), ("full window", dev)):
    with torch.cuda.stream(stream):
        for _ in range(3):
            dfcn.collect_window(*dfcn.enqueue_window(ctx, fs_seed("x"), header, famset, relu_ctx=relu_ctx))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pend = [dfcn.enqueue_window(ctx, fs_seed("x"), header, famset, relu_ctx=relu_ctx) for _ in range(K)]
        for c in (ctx, relu_ctx):
            ev = torch.cuda.Event()
            ev.record(c.stream)
            stream.wait_event(ev)
        e1.record(stream)
        torch.cuda.synchronize()
        for p in pend:
            dfcn.collect_window(*p)
    print(f"{label}: {e0.elapsed_time(e1) / K:.3f} ms per window")
