"""Host->device probe for the end-to-end leg: pinned H2D bandwidth and e2e window timing breakdown.

    python scripts/h2d_probe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    n = 1_591_869_440
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    for chunk in (n, 64 << 20):
        t0 = time.perf_counter()
        for o in range(0, n, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"H2D pinned chunk {chunk >> 20} MiB: {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)")
    hp = torch.empty(n, dtype=torch.uint8)   # pageable
    t0 = time.perf_counter()
    d.copy_(hp)
    torch.cuda.synchronize()
    print(f"H2D pageable: {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")

    from paper_2307_16273_b200 import api
    from paper_2307_16273_b200 import fcn as dfcn
    from synth import fcn
    from synth.prng import fs_seed
    fams = fcn.assemble_families(fcn.C4_SHAPE, fcn.generate_trace(fcn.C4_SHAPE))
    pin = lambda a: torch.from_numpy(a).pin_memory()
    host = [dfcn.DeviceFamily(f.name, "matmul", A=pin(f.A), B=pin(f.B), trans_a=f.transA, trans_b=f.transB)
            if hasattr(f, "A") else dfcn.DeviceFamily(f.name, "relu", Z=pin(f.Z), GA=pin(f.GA), Q=f.Q, R=f.R)
            for f in fams]
    for f in fams:
        nb = (f.A.nbytes + f.B.nbytes) if hasattr(f, "A") else (f.Z.nbytes + f.GA.nbytes)
        print(f"  {f.name}: {nb / 1e6:.1f} MB")
    stream = torch.cuda.Stream()
    ctx = api.Context(0, stream)
    cs = torch.cuda.Stream()
    hdr = fcn.fcn_header(fcn.C4_SHAPE)
    with torch.cuda.stream(stream):
        for i in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dfcn.prove_window_from_host(ctx, fs_seed("probe"), hdr, host, cs)
            torch.cuda.synchronize()
            print(f"e2e window {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms")
        dev = dfcn.upload_families(fams)
        torch.cuda.synchronize()
        for i in range(3):
            t0 = time.perf_counter()
            dfcn.prove_window(ctx, fs_seed("probe"), hdr, dev)
            torch.cuda.synchronize()
            print(f"resident window {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms")


if __name__ == "__main__":
    main()
