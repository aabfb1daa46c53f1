"""Timeline of the claim-chained C4 window (diagnostics): the bench's chained-window setup, one window
enqueued after two warm-ups, stage markers (chain.enqueue_window_chained(marks=...)) printed as ms since the
window's start.  Env CHAIN_MERGE_STREAMS / CHAIN_MERGE_BUDGET / CHAIN_MM_STREAMS as bench.py's flags."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2307_16273_b200 import api, build, chain
from synth import fcn
from synth.prng import fs_seed

build.build(verbose=False)
shape, fams, (top, ptens) = bench.c4_workload(0)
cfams, cts = chain.upload_plan(fams, ptens, device="cuda:0", top=top)
stream = torch.cuda.Stream()
ctx = api.Context(0, stream)
relu_ctx = api.Context(0, torch.cuda.Stream(priority=-1))
nmm = int(os.environ.get("CHAIN_MM_STREAMS", "8"))
mm_ctxs = [api.Context(0, torch.cuda.Stream()) for _ in range(nmm - 1)]
for c in [ctx] + mm_ctxs:
    c.set_sm_budget(max(8, 148 // nmm))
nms = int(os.environ.get("CHAIN_MERGE_STREAMS", "8"))
budget = int(os.environ.get("CHAIN_MERGE_BUDGET", "0")) or 148
mctxs = [api.Context(0, torch.cuda.Stream()) for _ in range(nms)]
for c in mctxs:
    c.set_sm_budget(max(4, budget // nms))
wctx = api.Context(0, torch.cuda.Stream())
rsctx = api.Context(0, torch.cuda.Stream()) if os.environ.get("CHAIN_RESCALE_STREAM", "1") != "0" else None
if rsctx is not None:
    rsctx.set_sm_budget(32)
    rsctx.set_persistent(os.environ.get("CHAIN_BESIDE_PERSIST", "0") == "1")
nl = int(os.environ.get("CHAIN_LATE_STREAMS", "4"))
after = os.environ.get("CHAIN_LATE_AFTER", "0") == "1"
lctxs = [api.Context(0, torch.cuda.Stream()) for _ in range(nl)]
for c in lctxs:
    c.set_sm_budget(max(2, 48 // max(1, nl)))
    c.set_persistent(os.environ.get("CHAIN_BESIDE_PERSIST", "0") == "1")
header = fcn.fcn_header(shape)
seed = fs_seed("C4-chained-rank0")
with torch.cuda.stream(stream):
    for _ in range(2):
        chain.prove_window_chained(ctx, seed, header, cfams, cts, relu_ctx=relu_ctx, mm_ctxs=mm_ctxs, wctx=wctx,
                                   merge_ctxs=mctxs, rescale_ctx=rsctx, late_ctxs=lctxs or None, late_after_relu=after)
    torch.cuda.synchronize()
    for rep in range(3):
        marks = []
        h = chain.enqueue_window_chained(ctx, seed, header, cfams, cts, relu_ctx=relu_ctx, mm_ctxs=mm_ctxs, wctx=wctx,
                                         merge_ctxs=mctxs, serial=True, marks=marks, rescale_ctx=rsctx, late_ctxs=lctxs or None, late_after_relu=after)
        chain.collect_window_chained(h)
        t0 = marks[0][2]
        print(f"--- window {rep} (merge streams {nms}, budget {budget}, mm streams {nmm}, rescale stream {rsctx is not None}, late streams {nl}, after relu {after})")
        if rep == 2 or os.environ.get("CHAIN_VERBOSE"):
            for label, st, ev in marks:
                print(f"  {t0.elapsed_time(ev):8.3f} ms  {label}")
        else:
            print(f"  end {t0.elapsed_time(marks[-1][2]):8.3f} ms")
