"""Sharded sumcheck host logic on CPU: world_size 2 over torch.distributed/gloo (-m "not gpu").

Each rank holds the slice of every table whose top index bit is its rank, runs
paper_2307_16273_b200.shard.prove with a CPU mock of the device session (tests/shard_mock.py), and
must end with the single-process oracle's transcript (claim, messages, challenges, finals, state) —
for several switch points of the gather-and-finish step.
"""
import os
import random
import socket

import pytest
import torch.multiprocessing as mp

from synth.prng import fs_seed, uniform_range

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2307_16273_b200 import shard
    from tests.shard_mock import MockSession
    comm = shard.TorchComm()
    out = []
    for (m, n_eq, K, switch, seedname, tabs, w) in cases:
        L = m - (world.bit_length() - 1)
        local = [t[rank << L:(rank + 1) << L] for t in tabs]
        sess = MockSession(oracle.Transcript(fs_seed(seedname)), m, n_eq, local, w, rank, world)
        res = shard.prove(sess, comm, switch_log=switch)
        out.append((res["claim"], res["msgs"], res["r"], res["finals"], res["state"]))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sumcheck_gloo_world2(oracle_lib):
    O = oracle_lib
    rng = random.Random(5)
    cases = []
    for (m, n_eq, K, switch) in [(5, 5, 2, 0), (5, 5, 2, 2), (6, 3, 2, 1), (6, 6, 3, 3), (4, 0, 1, 1), (6, 6, 2, 10)]:
        tabs = [[int(v) % P for v in uniform_range(11, 10 * m + k, (1 << m,), -(1 << 15), 1 << 15)] for k in range(K)]
        w = [rng.randrange(P) for _ in range(n_eq)]
        cases.append((m, n_eq, K, switch, f"shard-{m}-{n_eq}-{K}-{switch}", tabs, w))
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for ci, (m, n_eq, K, switch, seedname, tabs, w) in enumerate(cases):
        tr = O.Transcript(fs_seed(seedname))
        o = O.sumcheck_prove(tr, m, n_eq, tabs, w, None)
        for rank in range(world):
            claim, msgs, r, finals, state = results[rank][ci]
            assert claim == o["claim"] and msgs == o["msgs"] and r == o["r"] and finals == o["finals"], (ci, rank)
            assert state == tr.state()
