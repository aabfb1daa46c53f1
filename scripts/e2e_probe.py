"""e2e transport probe (under gpurun): the bench's C4 host stacks through fcn.upload_windows, with CUDA events
per window on the copy stream (DMA) and the widen stream.   python scripts/e2e_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_16273_b200 import build  # noqa: E402
from paper_2307_16273_b200 import fcn as dfcn  # noqa: E402


def main():
    build.build(verbose=False)
    shape, fams, tensors = bench.c4_workload(0)
    pinned = {}

    def pin(a):
        if id(a) not in pinned:
            small = a.size and int(a.max()) < (1 << 15) and int(a.min()) >= -(1 << 15)
            nz = np.flatnonzero(a.reshape(a.shape[0], -1).any(axis=1)) if a.ndim > 1 else np.array([0])
            n_real = int(nz[-1]) + 1 if nz.size else 1
            body = a[:n_real] if a.ndim > 1 else a
            t = torch.from_numpy(np.ascontiguousarray(body.astype(np.int16) if small else body)).pin_memory()
            pinned[id(a)] = dfcn.HostStack(t, a.shape) if (a.ndim > 1 and n_real < a.shape[0]) else t
        return pinned[id(a)]
    host = [dfcn.DeviceFamily(f.name, "matmul", A=pin(f.A), B=pin(f.B), trans_a=f.transA, trans_b=f.transB)
            if hasattr(f, "A") else dfcn.DeviceFamily(f.name, "relu", Z=pin(f.Z), GA=pin(f.GA), Q=f.Q, R=f.R) for f in fams]
    nbytes = sum(t.numel() * t.element_size() for t in pinned.values())
    for k, t in pinned.items():
        print(f"  stack {tuple(t.shape)} {t.dtype} pinned={t.data.is_pinned() if isinstance(t, dfcn.HostStack) else t.is_pinned()} "
              f"{t.numel() * t.element_size() / 1e6:.1f} MB")
    cs = torch.cuda.Stream()
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dfcn.upload_windows([host] * 5, cs, 0)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"upload_windows x5: {dt * 1e3:.2f} ms per window, {nbytes / dt / 1e9:.1f} GB/s")
    # raw: the same tensors copied with plain .to() on one stream
    flat = [t.data if isinstance(t, dfcn.HostStack) else t for t in pinned.values()]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(cs):
            outs = [[t.to("cuda", non_blocking=True) for t in flat] for _ in range(5)]
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 5
        print(f"plain .to() x5: {dt * 1e3:.2f} ms per window, {nbytes / dt / 1e9:.1f} GB/s")
        del outs


if __name__ == "__main__":
    main()
