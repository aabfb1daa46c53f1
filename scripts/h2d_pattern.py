"""H2D transport probe (under gpurun): one large pinned copy vs the per-stack copies of the e2e leg.
    python scripts/h2d_pattern.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch


def t_copy(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    n = 478_707_712
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    dt = t_copy(lambda: d.copy_(h, non_blocking=True))
    print(f"one copy {n / 1e6:.0f} MB: {dt * 1e3:.2f} ms = {n / dt / 1e9:.1f} GB/s")
    for parts in (4, 20, 64):
        c = n // parts

        def many():
            for i in range(parts):
                d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
        dt = t_copy(many)
        print(f"{parts} copies: {dt * 1e3:.2f} ms = {n / dt / 1e9:.1f} GB/s")

        def two_streams():
            for i in range(parts):
                with torch.cuda.stream(s1 if i % 2 else s2):
                    d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
        dt = t_copy(two_streams)
        print(f"{parts} copies on 2 streams: {dt * 1e3:.2f} ms = {n / dt / 1e9:.1f} GB/s")
    # allocation per copy (as .to(dev) does)
    c = n // 20

    def alloc_copies():
        out = [h[i * c:(i + 1) * c].to("cuda", non_blocking=True) for i in range(20)]
        return out
    dt = t_copy(alloc_copies)
    print(f"20 x .to(cuda) with allocation: {dt * 1e3:.2f} ms = {n / dt / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()


def uploader_probe():
    """The e2e leg's _Uploader on synthetic pinned stacks: int32 (copy only), int16 (copy + widen), HostStack."""
    from paper_2307_16273_b200 import fcn as dfcn
    dev = torch.device("cuda", 0)
    cs = torch.cuda.Stream()
    n = 24 << 20   # entries per stack
    kinds = {
        "int32": [torch.zeros(n, dtype=torch.int32).pin_memory() for _ in range(4)],
        "int16+widen": [torch.zeros(n, dtype=torch.int16).pin_memory() for _ in range(8)],
        "HostStack int16 (3/4 real)": [dfcn.HostStack(torch.zeros((12, n // 16), dtype=torch.int16).pin_memory(), (16, n // 16))
                                       for _ in range(8)],
    }
    for name, ts in kinds.items():
        nbytes = sum(t.numel() * t.element_size() for t in ts)

        def run():
            up = dfcn._Uploader(dev, cs)
            outs = [up.upload(t) for t in ts]
            torch.cuda.current_stream().wait_stream(up.ws)
            return outs
        dt = t_copy(run)
        print(f"_Uploader {name}: {nbytes / 1e6:.0f} MB in {dt * 1e3:.2f} ms = {nbytes / dt / 1e9:.1f} GB/s")


uploader_probe()
