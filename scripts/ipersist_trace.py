"""Per-round device timestamps of the persistent zkReLU rounds (ZKDL_IPERSIST_TRACE=1, printed by the library
to stderr) for one C4-size zkReLU (D = 2^23, Q = R = 16): workers, reduce, g + transcript, update."""
import os
import sys

os.environ["ZKDL_IPERSIST_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2307_16273_b200 import api
from synth.prng import fs_seed, uniform_range

logD = int(sys.argv[1]) if len(sys.argv) > 1 else 23
ctx = api.Context(0)
Z = torch.from_numpy(uniform_range(5, 1, (1 << logD,), -(1 << 31), 1 << 31)).cuda()
GA = torch.from_numpy(uniform_range(5, 2, (1 << logD,), -(1 << 31), 1 << 31)).cuda()
for rep in range(2):
    print(f"--- rep {rep}", file=sys.stderr)
    api.relu_prove(ctx, api.Transcript(ctx, fs_seed("trace")), Z, GA, 16, 16)
    torch.cuda.synchronize()
