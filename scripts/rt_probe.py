"""Tensor-core row dots vs the CUDA-core kernel (bit-exact), a few shapes; run under `timeout`."""
import random
import sys

import torch

sys.path.insert(0, ".")
from paper_2307_16273_b200 import api  # noqa: E402
from paper_2307_16273_b200._lib import lib  # noqa: E402

ctx = api.Context(0)
P = api.P
shapes = [(int(a), int(b)) for a, b in (x.split("x") for x in sys.argv[1:])] or [(1024, 8), (4096, 1024)]
for nrows, cols in shapes:
    M = torch.randint(-2 ** 31, 2 ** 31, (nrows, cols), dtype=torch.int64).to(torch.int32).cuda()
    pt = api._fr_buf([random.randrange(P) for _ in range(cols.bit_length() - 1)])
    outs = []
    for tc in (0, 1):
        o = torch.zeros((nrows, 32), dtype=torch.uint8, device="cuda")
        ctx.check(lib().zk_diag_rowdot(ctx.h, M.data_ptr(), nrows, cols, pt, o.data_ptr(), tc))
        outs.append(o.cpu())
    badrows = (outs[0] != outs[1]).any(dim=1).nonzero().flatten().tolist()
    tiles = sorted(set(r // 128 for r in badrows))
    print(f"rows {nrows} cols {cols}: mismatching rows {len(badrows)}, tiles {tiles[:20]}", flush=True)
