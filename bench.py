"""Benchmark of the zkDL prover hot path on B200 (contract: see DESIGN.md §7 "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

One step = one FAC4DNN proving window of the C4 workload (BASELINE.json metric: "prover s per
batch update (8-layer 10M FCN, bs 64)"): all 9 families (forward, input-gradient and
weight-gradient matmul families restricted and proved by the product sumcheck, and the stacked
zkReLU of 8 layers x 16 steps) under one Fiat-Shamir transcript, T' = 16 training steps per window.
value = seconds per batch update = window time / 16 (whole job: total time / total updates).
Under torchrun each rank proves its own window (weak scaling, no data-path collective).
The reference arm (--impl reference) times the CPU oracle on a bounded sample of the same window.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prover s per batch update (8-layer 10M FCN, bs 64); sumcheck Fr-mul/s vs peak"
UNIT = "s/update"
IMAD_LANES_PER_SM_CLK = 64          # fma pipe: rt_SMSP = 2 -> 16 lanes/clk/SMSP (B300_MICROARCH.md "Pipe rates")
IMAD_PER_FRMUL = 256                # CIOS 8x32-bit lower bound: 128 product + 128 reduction half-products


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    """SM clock / throttle-reason sampler for the timed region: NVML every 5 ms from a thread (the
    region can be ~100 ms, too short for nvidia-smi -lms), nvidia-smi as the fallback."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None
        self.nvml = None
        self.stop_flag = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _nvml_loop(self):
        pn = self.nvml
        while not self.stop_flag:
            try:
                sm = pn.nvmlDeviceGetClockInfo(self.h, pn.NVML_CLOCK_SM)
                rs = pn.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.nvml:
            self.stop_flag = False
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return
        self._start_smi()

    def _stop_nvml(self) -> dict:
        self.stop_flag = True
        self.thread.join(timeout=2)
        pn = self.nvml
        names = {"hw_slowdown": pn.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": pn.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": pn.nvmlClocksEventReasonSwThermalSlowdown,
                 "hw_power_brake": pn.nvmlClocksEventReasonHwPowerBrakeSlowdown,
                 "sw_power_cap": pn.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({nm for _, rs in self.rows for nm, bit in names.items() if rs & bit})
        sm = [float(s) for s, _ in self.rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(sm), "source": "nvml"}

    def _start_smi(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE, text=True)
        except Exception:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.rows.append([c.strip() for c in line.split(",")])
        self.thread = threading.Thread(target=rd, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        if self.nvml:
            return self._stop_nvml()
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) > 8:
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- distributed helpers
def dist_setup(n_gpus: int):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # ZKDL_BENCH_BACKEND=gloo: the multi-rank logic on fewer GPUs than ranks (tests; ranks share
        # devices round robin); the driver's runs use NCCL, one rank per GPU
        backend = os.environ.get("ZKDL_BENCH_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- workload
def c4_workload(rank: int):
    from synth import fcn
    from synth.prng import DATA_SEED
    t0 = time.time()
    trace = fcn.generate_trace(fcn.C4_SHAPE, seed=DATA_SEED + rank)
    fams = fcn.assemble_families(fcn.C4_SHAPE, trace)
    top = fcn.assemble_top_families(fcn.C4_SHAPE, trace, fams)
    tensors = fcn.plan_window(fcn.C4_SHAPE, trace, fams, top)
    log(f"[bench] rank {rank}: C4 trace + families generated in {time.time() - t0:.1f}s")
    return fcn.C4_SHAPE, fams, (top, tensors)


def family_bytes(fams) -> int:
    tot = 0
    for f in fams:
        tot += (f.A.nbytes + f.B.nbytes) if hasattr(f, "A") else (f.Z.nbytes + f.GA.nbytes)
    return tot


def frmul_model(fams, persist_log: int = 16, hb: int = 5) -> dict:
    """Algorithmic Fr-mul counts per window by kernel (DESIGN.md §6 counting model).  The split of the
    zkReLU i-rounds between the per-round kernel and the persistent one mirrors relu.cu (rounds with at
    most 2^persist_log pairs run in k_relu_ipersist; the last hb rounds in k_relu_itail)."""
    relu = [f for f in fams if not hasattr(f, "A")]
    out = {"k_relu_iround_f": 0, "k_relu_ipersist": 0, "k_sc_all": 0}
    for f in relu:
        D = f.Z.size
        logD = D.bit_length() - 1
        H = logD - min(hb, logD)
        t0 = next((t for t in range(1, H) if (D >> (t + 1)) <= (1 << persist_log)), H)
        # factored i-round, per pair (two sides), X = 1 derived from the per-term sums (ZKDL_IR_DERIVE, the
        # default): first round 2 x (T_a 1 + T_c 2 + T_b 4) = 14; folding rounds 2 x (3 fold + 1 + 4 + 4) = 24;
        # round 1 from the words (t0 >= 2, fold by byte tables) 2 x 9 = 18.  Explicit X = 1 (the persistent
        # rounds, ZKDL_IR_DERIVE=0): 18, 30, 24.  HI' products per thread and launch not counted.
        derive = os.environ.get("ZKDL_IR_DERIVE", "1") != "0"
        # the first round's linear terms from the Gram kernel's parity-split cells (relu.cu MODE bit 3; the
        # tensor-core bit sums run for logD >= 12, B >= 8): 2 x (T_b 4) = 8 products per pair
        cells = derive and os.environ.get("ZKDL_IR_CELLS", "1") != "0" and logD >= 12 and t0 >= 2
        for t in range(H):
            pairs = D >> (t + 1)
            if derive:   # the per-round and (round 2, later) the persistent rounds
                per = (8 if cells else 14) if t == 0 else (18 if t == 1 and t0 >= 2 else 24)
            else:
                per = 18 if t == 0 else (24 if t == 1 and t0 >= 2 else 30)
            out["k_relu_iround_f" if t < t0 else "k_relu_ipersist"] += per * pairs
    for f in fams:
        if hasattr(f, "A"):
            N = f.A.shape[0]
            D2 = f.A.shape[1] if f.transA else f.A.shape[2]
            # K = 2 product rounds: fold 4 + eq 1 + 3 evaluations x 2 = 11 per pair, pairs summed ~ N * D2
            out["k_sc_all"] += 11 * N * D2
    return out


def by_kernel(prof: dict) -> dict:
    """Merge template instantiations: {"k<true>": (n, ms), "k<false>": ...} -> {"k": (n, ms)}."""
    out = {}
    for k, (n, t) in prof.items():
        b = k.lstrip("(").split("<")[0]
        n0, t0 = out.get(b, (0, 0.0))
        out[b] = (n0 + n, t0 + t)
    return out


def dominant_kernel(prof: dict):
    """The kernel (all its instantiations) with the largest total duration."""
    g = by_kernel(prof)
    return max(g.items(), key=lambda kv: kv[1][1])[0] if g else None


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    import numpy as np
    import torch
    from paper_2307_16273_b200 import api, build
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    from synth.prng import fs_seed

    build.build(verbose=False)
    shape, fams, tensors = c4_workload(rank)
    in_bytes = family_bytes(fams)
    dev_fams = dfcn.upload_families(fams, device=f"cuda:{local}")
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=local)
    ctx = api.Context(local, stream)
    # zkReLU families on a second stream, concurrent with the matmul families (D3d transcripts)
    # the zkReLU family is the window's critical path: its stream gets the higher scheduling priority, so
    # the matmul families' CTAs fill the SMs it leaves idle instead of delaying it
    relu_ctx = api.Context(local, torch.cuda.Stream(device=local, priority=args.relu_priority)) if args.streams == 2 else None
    # matmul families spread over --mm-streams contexts (one stream each), persistent grids budgeted
    mm_ctxs = [api.Context(local, torch.cuda.Stream(device=local)) for _ in range(args.mm_streams - 1)]
    if args.mm_streams > 1:
        for c in [ctx] + mm_ctxs:
            c.set_sm_budget(args.mm_budget or max(8, 148 // args.mm_streams))
    ctxs = [ctx] + ([relu_ctx] if relu_ctx else []) + mm_ctxs
    # --pipeline: consecutive windows on alternating zkReLU and window-transcript streams, so a window's
    # zkReLU starts while the previous one finishes its latency-bound tail rounds (no cross-window waits)
    pipe = bool(args.pipeline) and relu_ctx is not None
    relu_ctxs = [relu_ctx] + ([api.Context(local, torch.cuda.Stream(device=local, priority=args.relu_priority))]
                              if pipe else [])
    wctxs = [api.Context(local, torch.cuda.Stream(device=local)) for _ in range(2)] if pipe else [None, None]
    ctxs = ctxs + relu_ctxs[1:] + [c for c in wctxs if c is not None]
    ctxs_all = ctxs
    header = fcn.fcn_header(shape)
    seed = fs_seed(f"C4-rank{rank}")

    def prof_on(name):
        for c in ctxs:
            c.profile_filter(name)
            c.profile(True)
            c.profile_read()

    def prof_off() -> dict:
        merged = {}
        for c in ctxs:
            for k, (n, t) in c.profile_read().items():
                n0, t0 = merged.get(k, (0, 0.0))
                merged[k] = (n0 + n, t0 + t)
            c.profile(False)
            c.profile_filter(None)
        return merged

    def profiled_pass():
        """K windows, one stream, CUDA events around every launch: the per-kernel table."""
        prof_on(None)
        for _ in range(args.steps):
            dfcn.enqueue_window(ctx, seed, header, dev_fams, merge_aux=args.merge_aux)
        torch.cuda.synchronize()
        return prof_off()

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            dfcn.collect_window(*dfcn.enqueue_window(ctx, seed, header, dev_fams, relu_ctx=relu_ctxs[i % len(relu_ctxs)],
                                                     mm_ctxs=mm_ctxs, merge_aux=args.merge_aux, wctx=wctxs[i % 2]))
        # one untimed rehearsal of the timed region's K windows in flight: the stream-ordered memory pool grows
        # to its high-water mark here (mapping fresh device memory costs the host up to ~0.1 s on a new box)
        for p_ in [dfcn.enqueue_window(ctx, seed, header, dev_fams, relu_ctx=relu_ctxs[i % len(relu_ctxs)],
                                       mm_ctxs=mm_ctxs, merge_aux=args.merge_aux, wctx=wctxs[i % 2])
                   for i in range(args.steps)]:
            dfcn.collect_window(*p_)
        torch.cuda.synchronize()
        # kernel table first (outside the timed region) -> the dominant kernel
        prof_table = profiled_pass() if args.prof == "dominant" else None
        dom_name = dominant_kernel(prof_table) if prof_table else None
        # ---- timed region: K windows, inputs resident in HBM (0.97 GB of stacks per window > 126 MB L2)
        clocks = Clocks(local)
        clocks.start()
        launches0 = sum(c.launches for c in ctxs)
        if args.prof in ("inline", "dominant"):
            # events around every launch ("inline") or only around the dominant kernel's launches
            prof_on(dom_name)
        barrier(world)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        pending = [dfcn.enqueue_window(ctx, seed, header, dev_fams, relu_ctx=relu_ctxs[i % len(relu_ctxs)],
                                       mm_ctxs=mm_ctxs, merge_aux=args.merge_aux, wctx=wctxs[i % 2])
                   for i in range(args.steps)]
        for c in ctxs_all:   # the region ends when every stream of every window has
            ev_ = torch.cuda.Event()
            ev_.record(c.stream)
            stream.wait_event(ev_)
        ev1.record(stream)
        torch.cuda.synchronize()
        for p_ in pending:   # outputs stay in HBM until here (outside the timed region)
            res = dfcn.collect_window(*p_)
        del pending
        barrier(world)
        launches = sum(c.launches for c in ctxs) - launches0
        clk = clocks.stop()
        prof_live = prof_off() if args.prof in ("inline", "dominant") else {}
        if args.prof == "inline":
            prof_table = prof_live
        elif args.prof == "separate":
            prof_table = profiled_pass()
            prof_live = prof_table
    prof = prof_table
    n1 = None
    if not args.merge_aux and not args.profile_mode:
        # SURVEY 8(f) N1 beside the headline: the same windows with every zkReLU family ending in the
        # aux-claim merge (D21), timed the same way
        with torch.cuda.stream(stream):
            dfcn.prove_window(ctx, seed, header, dev_fams, relu_ctx=relu_ctx, mm_ctxs=mm_ctxs, merge_aux=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pend = [dfcn.enqueue_window(ctx, seed, header, dev_fams, relu_ctx=relu_ctx, mm_ctxs=mm_ctxs, merge_aux=True)
                    for _ in range(args.steps)]
            e1.record(stream)
            torch.cuda.synchronize()
            del pend
        n1 = {"ms_per_step": max_over_ranks(e0.elapsed_time(e1), world) / args.steps,
              "what": "the same window with the zkReLU aux-claim merge (one aux claim per ReLU family)"}
    chained = None
    if not args.profile_mode and not args.no_chained:
        # SURVEY 8(f) N3 beside the headline: the claim-chained window (Protocol 1 lines 7-8, DESIGN.md
        # D25) -- matmul families, the claim merges that leave one claim per tensor family, the chained
        # zkReLU at the merged points and its aux merge -- timed the same way
        from paper_2307_16273_b200 import chain
        top, ptens = tensors
        cfams, cts = chain.upload_plan(fams, ptens, device=f"cuda:{local}", top=top)
        cseed = fs_seed(f"C4-chained-rank{rank}")
        # each window's transcript on its own stream (two alternate), so a window's matmul families and
        # merges overlap the previous window's zkReLU
        cwctxs = [api.Context(local, torch.cuda.Stream(device=local)) for _ in range(2)]
        # stage 2's claim merges (latency-bound sumchecks) side by side on budgeted streams
        mctxs = [api.Context(local, torch.cuda.Stream(device=local)) for _ in range(args.merge_streams)]
        for c in mctxs:   # the merges' persistent grids together leave room for the zkReLU's persistent
            # rounds of the previous window (k_relu_ipersist needs ~65 SMs co-resident; a cooperative launch
            # that cannot get them waits, and the window's critical path with it)
            c.set_sm_budget(max(4, (args.merge_budget or 148) // max(1, args.merge_streams)))
        # the top layer's rescale (+ its aux merge) beside the zkReLU on a stream of its own
        rsctx = api.Context(local, torch.cuda.Stream(device=local)) if args.rescale_stream else None
        if rsctx is not None:   # its persistent grids (k_sc_all: one SM per CTA) beside k_relu_ipersist (129
            # CTAs, two per SM): 2 x (148 - 32) >= 129, so neither can be left partly resident (no
            # spin-wait deadlock between the two)
            rsctx.set_sm_budget(32)
            rsctx.set_persistent(False)
        # the claim merges stage 3 does not wait for (D25 order), beside it: 4 streams x 12 SMs (+ the rescale's
        # 32 <= 148 - 65, the co-residency rule of chain.enqueue_window_chained)
        # stage 1 (the matmul families, latency-bound persistent sumchecks) alone on the GPU in serial windows: its
        # own --chain-mm-streams contexts, 148 SMs shared out
        nmm1 = max(1, args.chain_mm_streams)
        c1ctxs = [api.Context(local, torch.cuda.Stream(device=local)) for _ in range(nmm1)]
        for c in c1ctxs:
            c.set_sm_budget(max(4, 148 // nmm1))
        lctxs = [api.Context(local, torch.cuda.Stream(device=local)) for _ in range(args.late_streams)]
        for c in lctxs:   # per-round sumcheck launches beside the zkReLU: no spin-waiting grid of theirs can be
            # left partly resident behind the zkReLU stream's (higher-priority) CTAs
            c.set_sm_budget(max(2, 48 // max(1, args.late_streams)))
            c.set_persistent(False)
        streams_all = [c.stream for c in ctxs + cwctxs + mctxs + ([rsctx] if rsctx else []) + lctxs + c1ctxs]
        with torch.cuda.stream(stream):
            for i in range(2):
                chain.prove_window_chained(c1ctxs[0], cseed, header, cfams, cts, relu_ctx=relu_ctx, mm_ctxs=c1ctxs[1:],
                                           wctx=cwctxs[i % 2], merge_ctxs=mctxs, rescale_ctx=rsctx, late_ctxs=lctxs or None)
            torch.cuda.synchronize()
            # the kernel table of one window (every launch bracketed, outside the timed region)
            prof_on(None)
            for c in cwctxs:
                c.profile(True)
                c.profile_read()
            for c in mctxs + ([rsctx] if rsctx else []) + lctxs + c1ctxs:
                c.profile(True)
                c.profile_read()
            chain.prove_window_chained(c1ctxs[0], cseed, header, cfams, cts, relu_ctx=relu_ctx, mm_ctxs=c1ctxs[1:], wctx=cwctxs[0],
                                       merge_ctxs=mctxs, rescale_ctx=rsctx, late_ctxs=lctxs or None)
            ctab = prof_off()
            for c in cwctxs + mctxs + ([rsctx] if rsctx else []) + lctxs + c1ctxs:
                for k, v in c.profile_read().items():
                    n0, t0 = ctab.get(k, (0, 0.0))
                    ctab[k] = (n0 + v[0], t0 + v[1])
                c.profile(False)
            # untimed rehearsal of the K windows in flight (the memory pool's high-water mark, see above)
            for p_ in [chain.enqueue_window_chained(c1ctxs[0], cseed, header, cfams, cts, relu_ctx=relu_ctx,
                                                    mm_ctxs=c1ctxs[1:], wctx=cwctxs[i % 2], merge_ctxs=mctxs,
                                                    serial=bool(args.chain_serial), rescale_ctx=rsctx,
                                                    late_ctxs=lctxs or None) for i in range(args.steps)]:
                chain.collect_window_chained(p_)
            torch.cuda.synchronize()
            barrier(world)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            pend = [chain.enqueue_window_chained(c1ctxs[0], cseed, header, cfams, cts, relu_ctx=relu_ctx,
                                                 mm_ctxs=c1ctxs[1:],
                                                 wctx=cwctxs[i % 2], merge_ctxs=mctxs, serial=bool(args.chain_serial),
                                                 rescale_ctx=rsctx, late_ctxs=lctxs or None)
                    for i in range(args.steps)]
            for st in streams_all:   # the region ends when every stream of every window has
                ev = torch.cuda.Event()
                ev.record(st)
                stream.wait_event(ev)
            c1.record(stream)
            torch.cuda.synchronize()
            cres = None
            for p_ in pend:
                cres = chain.collect_window_chained(p_)
            del pend
        cms = max_over_ranks(c0.elapsed_time(c1), world) / args.steps
        cby = by_kernel(ctab)
        chained = {"ms_per_step": round(cms, 4), "s_per_update": cms / 1000.0 / shape.steps,
                   "merge_streams": args.merge_streams, "serial_windows": bool(args.chain_serial),
                   "rescale_stream": bool(args.rescale_stream), "late_merge_streams": args.late_streams,
                   "stage1_streams": nmm1,
                   "kernels_ms_one_window_serialised": {k: round(t, 4) for k, (n, t) in
                                                        sorted(cby.items(), key=lambda kv: -kv[1][1])[:14]},
                   "kernel_launches_one_window": {k: n for k, (n, t) in sorted(cby.items(), key=lambda kv: -kv[1][1])[:14]},
                   "launches_one_window": sum(n for n, t in cby.values()),
                   "claim_merges": sorted(cres["merges"]), "window_state": cres["window_state"].hex()[:16],
                   "what": "the claim-chained window (N3) with the top layer (N2): every matmul family and the "
                           "loss family, one claim merge per tensor family with several claims, the zkReLU at "
                           "the merged points + aux merge, the top-layer rescale + its aux merge; ends with one "
                           "claim per committed tensor family and one on each aux"}
        del cfams, cts
        torch.cuda.empty_cache()
    ms_local = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms_local, world)
    updates = world * args.steps * shape.steps
    value = (ms / 1000.0) / updates
    # ---- e2e: host (pinned) -> device copies of the window's inputs inside the timed region
    pinned = {}

    def pin(a):   # one pinned buffer per distinct stack (shared stacks are uploaded once per window); a stack
        # whose entries fit 16 bits (the matmul operands: X, W, A, G_Z) travels as int16 and is widened on
        # the device (zk_widen_i16): the same int32 tensor, half the PCIe bytes
        if id(a) not in pinned:
            small = args.e2e_i16 and a.size and int(a.max()) < (1 << 15) and int(a.min()) >= -(1 << 15)
            # trailing all-zero slots (the stack axis padded to a power of two) are zero-filled on the device
            nz = np.flatnonzero(a.reshape(a.shape[0], -1).any(axis=1)) if a.ndim > 1 else np.array([0])
            n_real = int(nz[-1]) + 1 if nz.size else 1
            body = a[:n_real] if a.ndim > 1 else a
            # a weight stack (slot = (step, layer)): the first step's slots + int8 differences to the same layer
            # one step earlier (SGD moves a weight by a few quantisation steps), rebuilt by zk_undelta_i8
            ds = dfcn.delta_stack(a, n_real) if (args.e2e_delta and small and a.ndim > 1) else None
            if ds is not None:
                pinned[id(a)] = ds
                return ds
            t = torch.from_numpy(np.ascontiguousarray(body.astype(np.int16) if small else body)).pin_memory()
            pinned[id(a)] = dfcn.HostStack(t, a.shape) if (a.ndim > 1 and n_real < a.shape[0]) else t
        return pinned[id(a)]

    host_fams = [dfcn.DeviceFamily(f.name, "matmul", A=pin(f.A), B=pin(f.B), trans_a=f.transA, trans_b=f.transB)
                 if hasattr(f, "A") else dfcn.DeviceFamily(f.name, "relu", Z=pin(f.Z), GA=pin(f.GA), Q=f.Q, R=f.R)
                 for f in fams]
    e2e_steps = 0 if args.profile_mode else max(1, args.steps)   # the same K windows as the device-timed value
    copy_stream = torch.cuda.Stream(device=local)
    with torch.cuda.stream(stream):
        for _ in range(2 if e2e_steps else 0):   # untimed warm-up with the timed call's shape: the caching
            # allocator then holds upload buffers for e2e_steps windows in flight (a cudaMalloc inside the
            # timed region synchronises the device and showed up as 20-60 ms outliers)
            dfcn.prove_windows_from_host(ctx, [(seed, header, host_fams)] * e2e_steps, copy_stream,
                                         relu_ctx=relu_ctx, mm_ctxs=mm_ctxs, merge_aux=args.merge_aux)
            torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        # pinned host -> HBM per family on a copy stream, each window's uploads behind the previous
        # window's and overlapped with its proofs; proof bytes come back to the host
        out = dfcn.prove_windows_from_host(ctx, [(seed, header, host_fams)] * e2e_steps, copy_stream,
                                           relu_ctx=relu_ctx, mm_ctxs=mm_ctxs, merge_aux=args.merge_aux)
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    uploads_ms = None
    if e2e_steps:   # the transport alone (same uploads, no proofs): what the e2e value is bound by
        with torch.cuda.stream(stream):
            dfcn.upload_windows([host_fams] * e2e_steps, copy_stream, local)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dfcn.upload_windows([host_fams] * e2e_steps, copy_stream, local)
            torch.cuda.synchronize()
            uploads_ms = 1e3 * (time.perf_counter() - t0) / e2e_steps
    h2d = sum(t.numel() * t.element_size() for t in pinned.values())   # distinct stacks (real slots), copied once each
    d2h = dfcn.window_out_bytes(dev_fams, bool(args.merge_aux)) + 4     # proofs, points, states + range flag
    e2e_value = e2e_s / (world * e2e_steps * shape.steps) if e2e_steps else None
    # ---- roofline of the dominant kernel (live CUDA-event durations over the timed region)
    per_step = {k: (n / args.steps, t / args.steps) for k, (n, t) in prof.items()}
    total_kernel_ms = sum(t for _, t in per_step.values())
    dom_name = dominant_kernel(prof) or "none"
    prof_live = by_kernel(prof_live)
    live = prof_live.get(dom_name, (0, 0.0))   # the dominant kernel's launches inside the timed region
    dom_launches, dom_ms = live[0] / args.steps, live[1] / args.steps
    model = frmul_model(fams)
    clock_mhz = clk.get("sm_max_mhz") or 1965.0
    imad_peak = 148 * IMAD_LANES_PER_SM_CLK * clock_mhz * 1e6             # lane-IMAD/s
    frmul_peak = imad_peak / IMAD_PER_FRMUL
    rf = None
    key = next((k for k in model if dom_name.startswith(k) or k in dom_name), None)
    if key and dom_ms > 0:
        achieved = model[key] / (dom_ms / 1000.0) / 1e9
        rf = {"bound": "alu", "kernel": dom_name, "achieved": round(achieved, 3), "peak": round(frmul_peak / 1e9, 3),
              "unit": "GFr-mul/s", "frac": round(achieved / (frmul_peak / 1e9), 4), "traffic": None,
              "peak_basis": f"148 SM x {IMAD_LANES_PER_SM_CLK} IMAD lanes/clk x {clock_mhz:.0f} MHz / {IMAD_PER_FRMUL} IMAD per Fr-mul",
              "ms_per_step": round(dom_ms, 4), "share_of_step": round(dom_ms / ms_local * args.steps, 4)}
    else:
        rf = {"bound": "alu", "kernel": dom_name, "achieved": None, "peak": round(frmul_peak / 1e9, 3),
              "unit": "GFr-mul/s", "frac": None, "traffic": None, "ms_per_step": round(dom_ms, 4),
              "share_of_step": round(dom_ms / ms_local * args.steps, 4) if ms_local else None}
    rf["launches_per_step"] = dom_launches
    try:   # the committed product-rate measurements (profiles/r2/frmul_peaks.json) as second denominators
        pk = json.load(open(os.path.join(ROOT, "profiles", "r2", "frmul_peaks.json")))
        if rf.get("achieved"):
            meas = pk["products_per_s"]["fp64_pipe_product"] / 1e9
            ana = pk["analytic_bounds_per_s"]["fp64_product_issue"]["value"] / 1e9
            rf["frac_of_measured_product_rate"] = round(rf["achieved"] / meas, 4)
            rf["frac_of_fp64_product_issue_bound"] = round(rf["achieved"] / ana, 4)
            rf["measured_peaks_basis"] = ("profiles/r2/frmul_peaks.json: the kernel's product (FP64 pipe, fr64.cuh) "
                                          f"register-resident {meas:.1f} G/s measured; its issue bound {ana:.1f} G/s; "
                                          "'peak' stays the IMAD-pipe bound of the north star's wording")
    except (OSError, ValueError, KeyError):
        pass
    try:   # DRAM traffic of the dominant kernel's captured launch (ncu --set full, committed under profiles/)
        tj = json.load(open(os.path.join(ROOT, "profiles", "r2", "ncu_traffic_r2.json")))
        base = dom_name.split("<")[0]
        if base in tj:
            L0 = tj[base]["launches"][0]
            rf["traffic"] = L0["dram_read"] + L0["dram_write"]
            rf["traffic_note"] = (f"bytes of one captured launch ({L0['launch']}) against {L0['algorithmic']} "
                                  f"algorithmic bytes ({L0['algorithmic_note']}); {tj['source']}")
    except (OSError, ValueError, KeyError):
        pass
    rf["durations"] = {
        "dominant": "CUDA events on the launch stream around each launch of this kernel only, inside the timed "
                    "region; the kernel table comes from an identical K-window pass with every launch bracketed",
        "inline": "CUDA events around every launch on the launch stream, inside the timed region",
        "separate": "CUDA events around every launch, second identical K-window pass after the timed region",
    }[args.prof]
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "fr_bls12_381 (8x32-bit Montgomery)", "data": "synthetic (seeded quantized FCN training trace)",
        "config": {"workload": "C4: FAC4DNN window of the 3072(->4096)-1024x8-10(->16) FCN, batch 64, T'=16 steps, "
                               "9 families (F x3, GA x2, GW x3, ReLU D=2^23), one transcript",
                   "updates_per_step": shape.steps, "input_bytes_per_step": in_bytes,
                   "l2": "inputs larger than L2 (0.97 GB of distinct stacks, 1.59 GB of family operands read per window, vs 126 MB)", "parallelism": f"replica x{world}", "streams": args.streams, "mm_streams": args.mm_streams, "pipelined_windows": pipe, "mm_budget": args.mm_budget or max(8, 148 // args.mm_streams), "relu_aux_merge": bool(args.merge_aux)},
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "fcn.prove_windows_from_host: pinned host stacks (16-bit stacks as int16, weight stacks as "
                        "their first step + int8 step differences, rebuilt on the device) -> HBM per family on a copy stream "
                        "(shared stacks once per window), each window's uploads behind the previous window's and "
                        "overlapped with the proofs; proofs back to the host", "windows": e2e_steps,
                "uploads_alone_ms_per_window": None if uploads_ms is None else round(uploads_ms, 3)},
        "roofline": rf,
        "n1_relu_aux_merge": n1,
        "n3_chained_window": chained,
        "kernels_ms_per_step": {k: round(t, 4) for k, (n, t) in sorted(per_step.items(), key=lambda kv: -kv[1][1])[:16]},
        "kernel_launches_per_step": {k: n for k, (n, t) in sorted(per_step.items(), key=lambda kv: -kv[1][1])[:16]},
        "kernel_ms_total_per_step": round(total_kernel_ms, 4),
        "clocks": clk,
        "paper_context": {"value": 0.84, "unit": "s/update", "hardware": "A100", "note": "PT/step at T'=16, BS 64 (PAPER.md L405); includes commitments, not this metric"},
    }
    if not args.no_c5 and not args.profile_mode:
        # BASELINE configs[4] alongside: one 2^26 sumcheck sharded over the same ranks (strong scaling)
        try:
            with torch.cuda.stream(stream):
                c5 = c5_measure(ctx, rank, world, 26, 3, 1)
            peak = 148 * IMAD_LANES_PER_SM_CLK * clock_mhz * 1e6 / IMAD_PER_FRMUL / 1e9
            out["c5_sharded"] = {"m": 26, "G": world, "ms_per_proof": c5["ms"], "frmul_per_s": c5["frmul_per_s"],
                                 "frac_of_frmul_peak": round(c5["frmul_per_s"] / 1e9 / peak, 4), "scaling": "strong",
                                 "proof_digest": c5["digest"], "note": "whole-proof rate incl. transcript steps and "
                                 "(G > 1) NCCL all-gathers; bench.py --config C5 gives the kernel table"}
        except Exception as e:   # never lose the headline line to the auxiliary measurement
            out["c5_sharded"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_mode:
        with torch.cuda.stream(stream):
            gfull = gpu_full_families(ctx, dev_fams, FULL_FAMILIES)
        out["cpu_baseline"] = cpu_baseline(fams, shape, sample_scale=args.cpu_sample, gpu_full_ms=round(gfull, 4))
    if rank == 0:
        print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- C5: one (sharded) 2^m product sumcheck
def c5_frmul_model(m: int, tail_log: int = 16, hb: int = 5) -> dict:
    """Algorithmic Fr-mul count of one C5 proof (K = 2, n_eq = m) by kernel, mirroring
    sumcheck.cu: round 0 (k_sc_round0_int, grouped eq weights): no Fr product per pair -- three exact
    integer multiply-accumulates E' x (P + 2^64) into 352-bit accumulators, reduced once per CTA and
    group ("int_mac_per_pair"); round 1 (k_sc_round2f folding from int32): 4 folds, each two 32 x 256-bit
    multiply-accumulates and one reduction (3/4 of a product) + E' a (2) + 3 = 8; folding rounds: fold 4 + 2 + 3 = 9 (plus one HI product
    per pair where the groups are too small, "flat"); the last rounds (<= 2^tail_log entries after the
    fold) in k_sc_all: fold 4 + eq 1 + 3 x 2 = 11 per pair (7 in the last, eq-free round).  With f(1) derived
    from the running claim (ZKDL_SC_DERIVE, the default) the folding rounds of k_sc_round2f skip one product:
    round 1 7, folding rounds 8."""
    derive = os.environ.get("ZKDL_SC_DERIVE", "1") != "0"
    out = {"k_sc_round2f": 0, "k_sc_all": 0, "k_sc_round0_int": 0}
    int0 = False
    for t in range(m):
        pairs = 1 << (m - t - 1)
        if t >= 1 and m - t <= tail_log:
            has_e = 1 if t + 1 < m else 0
            out["k_sc_all"] += pairs * (4 + has_e + 3 * (1 + has_e))
            continue
        nv = m - t - 1                      # eq variables of the pair index
        hbe = min(m - 1, hb)
        flat = nv > hbe and nv - hbe < 10    # LO x HI with groups < 1024 pairs: per-pair HI product
        if t == 0 and nv > hbe and not flat:
            out["int_mac_per_pair"] = 3
            int0 = True
            continue
        per = 7 if t == 0 else (8 if t == 1 and int0 else 9) - (1 if derive and t >= 1 else 0)
        out["k_sc_round2f"] += pairs * (per + (1 if flat else 0))
    out["total"] = out["k_sc_round2f"] + out["k_sc_all"]
    return out


def c5_measure(ctx, rank: int, world: int, m: int, steps: int, warmup: int, switch_log: int = 12) -> dict:
    """Time the C5 statement sum_x eq(w, x) A(x) B(x) over 2^m entries (D3c: "c5/hdr", w drawn from the
    transcript, claim computed in round 0), sharded over the `world` ranks on its last-bound variables
    (D19; G = 1: the single-device prover).  Inputs: int32 slices generated on the device, resident
    before the timed region; every step proves from a fresh transcript."""
    import torch
    from paper_2307_16273_b200 import api, shard
    from synth.prng import DATA_SEED, fs_seed, uniform_range_torch
    dev = torch.device("cuda", ctx.device)
    s = world.bit_length() - 1
    n_loc = 1 << (m - s)
    A = uniform_range_torch(DATA_SEED, 21, n_loc, -(1 << 15), 1 << 15, dev, offset=rank * n_loc)
    B = uniform_range_torch(DATA_SEED, 22, n_loc, -(1 << 15), 1 << 15, dev, offset=rank * n_loc)
    if world > 1:   # the exchange owned by the library: one NCCL communicator per context
        shard.attach_nccl(ctx)
    torch.cuda.synchronize()

    def one():
        tr = api.Transcript(ctx, fs_seed(f"C5-m{m}"))
        tr.absorb("c5/hdr", m.to_bytes(4, "little"))
        w = tr.challenges("c5/w", m)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        if world == 1:
            res = api.sumcheck_prove(ctx, tr, m, m, [A, B], w)
        else:
            sess = shard.ShardSession(ctx, tr, m, m, [A, B], w, rank, world)
            res = shard.prove_nccl(sess, switch_log=switch_log)
            sess.close()
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        tr.close()
        return e0.elapsed_time(e1), res

    for _ in range(warmup):
        one()
    times = []
    res = None
    for _ in range(steps):
        ms, res = one()
        times.append(max_over_ranks(ms, world))
    ms = statistics.median(times)
    model = c5_frmul_model(m)
    frmul = model["total"]
    return {"m": m, "G": world, "ms": round(ms, 4), "ms_min": round(min(times), 4), "frmul": frmul, "model": model,
            "frmul_per_s": frmul / (ms / 1000.0), "digest": __import__("hashlib").sha256(res["proof"]).hexdigest()[:16]}


def run_c5(args, rank, world, local):
    """--config C5: the sharded single sumcheck (BASELINE configs[4]), strong scaling."""
    import torch
    from paper_2307_16273_b200 import api, build
    build.build(verbose=False)
    stream = torch.cuda.Stream(device=local)
    ctx = api.Context(local, stream)
    with torch.cuda.stream(stream):
        clocks = Clocks(local)
        clocks.start()
        r = c5_measure(ctx, rank, world, args.c5_log, args.steps, args.warmup)
        clk = clocks.stop()
        prof = {}
        if world == 1:   # per-kernel table of one more proof (every launch bracketed)
            ctx.profile(True)
            ctx.profile_read()
            c5_measure(ctx, rank, world, args.c5_log, 1, 0)
            prof = by_kernel(ctx.profile_read())
            ctx.profile(False)
    clock_mhz = clk.get("sm_max_mhz") or 1965.0
    peak = 148 * IMAD_LANES_PER_SM_CLK * clock_mhz * 1e6 / IMAD_PER_FRMUL / 1e9
    rf = None
    if prof:
        n, kms = prof.get("k_sc_round2f", (0, 0.0))
        if kms > 0:
            ach = r["model"]["k_sc_round2f"] / (kms / 1000.0) / 1e9
            rf = {"bound": "alu", "kernel": "k_sc_round2f", "achieved": round(ach, 3), "peak": round(peak, 3),
                  "unit": "GFr-mul/s", "frac": round(ach / peak, 4), "traffic": None, "launches_per_proof": n,
                  "ms_per_proof": round(kms, 4), "share_of_step": round(kms / r["ms"], 4),
                  "durations": "CUDA events around every launch of one more proof after the timed region"}
            try:   # DRAM traffic of a captured launch at m = 26 (ncu --set full, committed under profiles/)
                L0 = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic_r1j.json")))["k_sc_round2f"]["launches"][0]
                if args.c5_log == 26:
                    rf["traffic"] = L0["dram_read"] + L0["dram_write"]
                    rf["traffic_note"] = (f"bytes of one captured launch ({L0['launch']}) against {L0['algorithmic']} "
                                          f"algorithmic bytes ({L0['algorithmic_note']})")
            except (OSError, ValueError, KeyError):
                pass
    out = {"metric": f"C5 sharded sumcheck: prover s per 2^{args.c5_log} product sumcheck (K=2, eq over all variables)",
           "value": r["ms"] / 1000.0, "unit": "s/proof", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": r["ms"], "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
           "dtype": "fr_bls12_381 (8x32-bit Montgomery)", "data": "synthetic (A, B ~ U[-2^15, 2^15) int32, counter PRNG)",
           "config": {"workload": f"C5: sum_x eq(w,x) A(x) B(x), 2^{args.c5_log} entries, sharded on the last-bound variables over G={world}",
                      "m": args.c5_log, "parallelism": f"shard x{world}", "l2": "inputs larger than L2" if args.c5_log >= 24 else "inputs fit L2"},
           "frmul_per_s": r["frmul_per_s"], "frmul_per_proof": r["frmul"], "proof_digest": r["digest"],
           "roofline": rf, "kernels_ms_per_step": {k: round(t, 4) for k, (n, t) in sorted(prof.items(), key=lambda kv: -kv[1][1])[:12]},
           "clocks": clk}
    if rank == 0:
        print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- T' x BS sweep (SURVEY §8(f) N3's workload)
def run_sweep(args, rank, world, local):
    """--config sweep: the C4 network at T' in --sweep-T and BS in --sweep-BS, one line with per-update
    proving time and per-update sumcheck proof bytes per point -- the shape of the paper's Table 1
    (PT and PS per step fall with T' until they plateau), for this hot path only (no
    commitments, so CS and the commitment part of PS are not comparable)."""
    import dataclasses

    import torch
    from paper_2307_16273_b200 import api, build
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    from synth.prng import DATA_SEED, fs_seed
    build.build(verbose=False)
    stream = torch.cuda.Stream(device=local)
    ctx = api.Context(local, stream)
    relu_ctx = api.Context(local, torch.cuda.Stream(device=local))
    mm = [api.Context(local, torch.cuda.Stream(device=local))]
    for c in [ctx] + mm:
        c.set_sm_budget(37)
    rows = []
    for T in args.sweep_T:
        for bs in args.sweep_BS:
            shape = dataclasses.replace(fcn.C4_SHAPE, name=f"C4-T{T}-BS{bs}", batch=bs, steps=T)
            t0 = time.time()
            fams = fcn.assemble_families(shape, fcn.generate_trace(shape, seed=DATA_SEED + rank))
            gen_s = time.time() - t0
            dev_fams = dfcn.upload_families(fams, device=f"cuda:{local}")
            header = fcn.fcn_header(shape)
            seed = fs_seed(shape.name)
            with torch.cuda.stream(stream):
                res = dfcn.prove_window(ctx, seed, header, dev_fams, relu_ctx=relu_ctx, mm_ctxs=mm)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                pend = [dfcn.enqueue_window(ctx, seed, header, dev_fams, relu_ctx=relu_ctx, mm_ctxs=mm)
                        for _ in range(args.steps)]
                e1.record(stream)
                torch.cuda.synchronize()
                del pend
            ms = max_over_ranks(e0.elapsed_time(e1), world) / args.steps
            proof_bytes = sum(len(r["proof"]) for r in res)
            rows.append({"T": T, "BS": bs, "s_per_update": ms / 1000.0 / T, "ms_per_window": round(ms, 3),
                         "proof_kB_per_update": round(proof_bytes / 1024.0 / T, 3),
                         "families": len(fams), "trace_gen_s": round(gen_s, 1)})
            log(f"[sweep] T'={T} BS={bs}: {ms / T:.3f} ms/update, {proof_bytes / 1024 / T:.2f} kB/update")
            del dev_fams, fams
            torch.cuda.empty_cache()
    out = {"metric": "prover s per batch update vs T' (aggregated steps) and BS (Table 1 shape, hot path only)",
           "value": rows[-1]["s_per_update"] if rows else None, "unit": "s/update", "n_gpus": world,
           "steps": args.steps, "warmup": 1, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
           "dtype": "fr_bls12_381 (8x32-bit Montgomery)", "data": "synthetic (seeded quantized FCN training trace)",
           "config": {"workload": "C4 network (3072(->4096)-1024x8-10(->16)) at each (T', BS)", "sweep": rows},
           "paper_context": {"table": "P:L391-416", "PT_s_per_step_A100": {"1": 6.2, "4": 1.9, "16": 0.84, "64": 0.85},
                             "note": "paper PT includes commitments and openings (excluded here)"}}
    if rank == 0:
        print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- N2: Protocol 2's zero form
def run_hadamard(args, rank, world, local):
    """--config hadamard: Protocol 2's zero form for the aggregated Hadamard product (SURVEY §8(f) N2,
    DESIGN.md D22): 0 = sum_x beta(w, x) (Y - A B) over 2^m entries, A, B ~ U[-2^15, 2^15), Y = A (.) B."""
    import torch
    from paper_2307_16273_b200 import api, build
    from synth.prng import DATA_SEED, fs_seed, uniform_range_torch
    build.build(verbose=False)
    stream = torch.cuda.Stream(device=local)
    ctx = api.Context(local, stream)
    m = args.c5_log
    dev = torch.device("cuda", local)
    A = uniform_range_torch(DATA_SEED, 21, 1 << m, -(1 << 15), 1 << 15, dev)
    B = uniform_range_torch(DATA_SEED, 22, 1 << m, -(1 << 15), 1 << 15, dev)
    Y = (A.to(torch.int64) * B.to(torch.int64)).to(torch.int32)
    times = []
    with torch.cuda.stream(stream):
        for i in range(args.warmup + args.steps):
            tr = api.Transcript(ctx, fs_seed(f"HD-m{m}"))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g = api.hadamard_zero_prove(ctx, tr, Y, A, B)
            e1.record(stream)
            torch.cuda.synchronize()
            tr.close()
            if i >= args.warmup:
                times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    first_ok = ((1 - g["w"][0]) * g["msgs"][0][0] + g["w"][0] * g["msgs"][0][1]) % 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001 == 0
    out = {"metric": f"N2: prover s per 2^{m} aggregated Hadamard product, Protocol 2 zero form", "value": ms / 1000.0,
           "unit": "s/proof", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
           "dtype": "fr_bls12_381 (8x32-bit Montgomery)", "data": "synthetic (A, B ~ U[-2^15, 2^15), Y = A B)",
           "config": {"workload": f"0 = sum_x beta(w,x) (Y - A B), 2^{m} entries", "m": m},
           "frmul_per_pair_model": "fold 6 + eq 1 + 3 x 2 = 13", "first_round_identity_holds": first_ok}
    if rank == 0:
        print(json.dumps(out), flush=True)


# ---------------------------------------------------------------- oracle (CPU) arm
def oracle_window_sample(fams, shape, frac_inst: int, relu_instances: int):
    """Time the oracle on a sub-stack of every family; return (seconds for the full window, sample note)."""
    import numpy as np
    import oracle as O
    from synth.fcn import fcn_header
    from synth.prng import fs_seed
    tr = O.Transcript(fs_seed("C4-oracle-sample"))
    tr.absorb("fcn/hdr", fcn_header(shape))
    est = 0.0
    parts = []
    for f in fams:
        tr.absorb("fcn/fam", f.name.encode())
        if hasattr(f, "A"):
            N = f.A.shape[0]
            n = max(1, N // frac_inst)
            t0 = time.perf_counter()
            O.matmul_prove(tr, np.ascontiguousarray(f.A[:n]), np.ascontiguousarray(f.B[:n]), f.transA, f.transB)
            dt = time.perf_counter() - t0
            est += dt * N / n
            parts.append(f"{f.name}:{n}/{N}")
        else:
            per = shape.batch * 1024
            n = relu_instances
            D = f.Z.size
            t0 = time.perf_counter()
            O.relu_prove(tr, np.ascontiguousarray(f.Z[:n * per]), np.ascontiguousarray(f.GA[:n * per]), f.Q, f.R)
            dt = time.perf_counter() - t0
            est += dt * D / (n * per)
            parts.append(f"{f.name}:{n}/{D // per}")
    return est, "oracle on sub-stacks " + ", ".join(parts) + " (time scaled linearly in the instance count)"


def oracle_full_families(fams, names):
    """The oracle on complete families (every instance, nothing extrapolated): seconds."""
    import numpy as np
    import oracle as O
    from synth.prng import fs_seed
    t0 = time.perf_counter()
    for f in fams:
        if f.name in names:
            O.matmul_prove(O.Transcript(fs_seed("C4-oracle-full-" + f.name)), np.ascontiguousarray(f.A),
                           np.ascontiguousarray(f.B), f.transA, f.transB)
    return time.perf_counter() - t0


def gpu_full_families(ctx, dev_fams, names, reps: int = 5) -> float:
    """The same complete families on the GPU (zk_matmul_prove, one stream, CUDA events): ms per pass."""
    import torch
    from paper_2307_16273_b200 import api
    from synth.prng import fs_seed
    sel = [f for f in dev_fams if f.name in names]

    def once():
        for f in sel:
            api.matmul_prove(ctx, api.Transcript(ctx, fs_seed("C4-oracle-full-" + f.name)), f.A, f.B, f.trans_a, f.trans_b)
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(reps):
        once()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


FULL_FAMILIES = ("F[9]", "GA[8]")   # two complete families of the C4 window (16 instances each)


def cpu_baseline(fams, shape, sample_scale: int = 16, gpu_full_ms: float | None = None):
    import oracle as O
    cores = len(os.sched_getaffinity(0))
    O.set_threads(cores)
    t0 = time.perf_counter()
    est, note = oracle_window_sample(fams, shape, frac_inst=sample_scale, relu_instances=4)
    wall = time.perf_counter() - t0
    full_all = oracle_full_families(fams, FULL_FAMILIES)
    O.set_threads(1)
    t1 = time.perf_counter()
    est1, note1 = oracle_window_sample(fams, shape, frac_inst=4 * sample_scale, relu_instances=1)
    wall1 = time.perf_counter() - t1
    full_one = oracle_full_families(fams, FULL_FAMILIES)
    O.set_threads(cores)
    return {"value": est / shape.steps, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": note + f"; sample wall {wall:.1f}s",
            "threads_1": {"value": est1 / shape.steps, "unit": UNIT, "cores": 1,
                          "sample": note1 + f"; sample wall {wall1:.1f}s"},
            "unextrapolated": {"families": list(FULL_FAMILIES), "what": "complete families of the window, every "
                               "instance proved by the oracle, nothing scaled", "s_all_cores": round(full_all, 4),
                               "s_1_thread": round(full_one, 4), "gpu_ms": gpu_full_ms,
                               "gpu_note": "the same families through zk_matmul_prove on one stream (CUDA events)"}}


def run_reference(args, rank, world, local):
    if rank != 0:
        return
    import oracle as O
    shape, fams, _ = c4_workload(0)
    cores = len(os.sched_getaffinity(0))
    O.set_threads(cores)
    for _ in range(args.warmup):
        oracle_window_sample(fams, shape, frac_inst=64, relu_instances=1)
    ests, walls = [], []
    t0 = time.perf_counter()
    note = ""
    for _ in range(args.steps):
        ts = time.perf_counter()
        est, note = oracle_window_sample(fams, shape, frac_inst=64, relu_instances=1)
        walls.append(time.perf_counter() - ts)
        ests.append(est)
    wall = time.perf_counter() - t0
    value = statistics.mean(ests) / shape.steps
    # ms_per_step is the measured time of one step (the bounded sample), so steps x ms_per_step is the run's
    # wall clock; value scales the sample to the whole window (every family's instance count, linear)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(walls), "higher_is_better": False,
           "value_basis": {"sample_ms_per_step": round(1000 * statistics.mean(walls), 1),
                           "window_ms_scaled": round(1000 * statistics.mean(ests), 1),
                           "scale": "each family's sampled instances scaled linearly to its full instance count; "
                                    "value = scaled window time / 16 updates"},
           "scaling": "weak", "vs_baseline": None, "dtype": "fr_bls12_381 (4x64-bit Montgomery, CPU)",
           "data": "synthetic (seeded quantized FCN training trace)",
           "config": {"workload": "C4: FAC4DNN window of the 3072(->4096)-1024x8-10(->16) FCN, batch 64, T'=16 steps",
                      "updates_per_step": shape.steps, "parallelism": f"cpu x{O.threads()}"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.threads(), "kind": "oracle",
                            "sample": note + f"; {args.steps} samples in {wall:.1f}s"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C4", "C5", "sweep", "hadamard"])
    ap.add_argument("--sweep-T", type=int, nargs="+", default=[1, 4, 16, 64])
    ap.add_argument("--sweep-BS", type=int, nargs="+", default=[16, 32, 64])
    ap.add_argument("--c5-log", type=int, default=26, help="C5: log2 m of the 2^m hypercube (22..30)")
    ap.add_argument("--no-c5", action="store_true", help="C4 line without the embedded C5 measurement")
    ap.add_argument("--no-chained", action="store_true", help="C4 line without the chained-window (N3) measurement")
    ap.add_argument("--chain-mm-streams", type=int, default=8,
                    help="chained window: streams (and SM budgets 148 / n) of stage 1's matmul families")
    ap.add_argument("--late-streams", type=int, default=4,
                    help="chained window: streams of the claim merges that prove beside stage 3 (0: after it)")
    ap.add_argument("--rescale-stream", type=int, default=1,
                    help="chained window: 1 = the top layer's rescale on its own stream, beside the zkReLU")
    ap.add_argument("--merge-streams", type=int, default=8, help="chained window: streams for the claim merges")
    ap.add_argument("--pipeline", type=int, default=0, choices=[0, 1],
                    help="1: consecutive windows on alternating zkReLU / transcript streams (measured 171 ms per "
                         "window against 11.2: two windows' persistent spin-waiting kernels interleave on the SMs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-delta", type=int, default=1, choices=[0, 1],
                    help="1: e2e ships weight stacks as their first step + int8 step-to-step differences (zk_undelta_i8)")
    ap.add_argument("--e2e-i16", type=int, default=1, choices=[0, 1],
                    help="1: e2e uploads stacks whose entries fit 16 bits as int16 (widened on the device)")
    ap.add_argument("--streams", type=int, default=2, choices=[1, 2],
                    help="2: zkReLU families on a second stream, concurrent with the matmul families")
    ap.add_argument("--mm-streams", type=int, default=2,
                    help="streams (contexts) the matmul families are spread over, side by side")
    ap.add_argument("--merge-aux", type=int, default=0, choices=[0, 1],
                    help="1: every zkReLU family ends with the aux-claim merge (P:L470, DESIGN.md D21)")
    ap.add_argument("--chain-serial", type=int, default=1, choices=[0, 1],
                    help="chained window: 1 = each window starts after the previous window's zkReLU stage (no "
                         "cross-window overlap: overlapping windows stalled on co-residency in some runs)")
    ap.add_argument("--merge-budget", type=int, default=0,
                    help="chained window: total SM budget of the claim merges' persistent grids (0: 148)")
    ap.add_argument("--relu-priority", type=int, default=-1, help="CUDA stream priority of the zkReLU stream (lower = higher)")
    ap.add_argument("--mm-budget", type=int, default=37,
                    help="SM budget of each matmul stream's persistent sumcheck grid (0: 148 / mm-streams)")
    ap.add_argument("--prof", default="dominant", choices=["dominant", "inline", "separate"],
                    help="where per-kernel CUDA-event durations come from (see roofline.durations)")
    ap.add_argument("--profile-mode", action="store_true", help="skip e2e and cpu_baseline (for ncu runs)")
    ap.add_argument("--cpu-sample", type=int, default=4, help="sub-stack divisor for the cpu_baseline sample")
    args = ap.parse_args()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, rank, 1, 0)
        return
    rank, world, local = dist_setup(args.gpus)
    if args.config == "C5":
        run_c5(args, rank, world, local)
    elif args.config == "sweep":
        run_sweep(args, rank, world, local)
    elif args.config == "hadamard":
        run_hadamard(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
