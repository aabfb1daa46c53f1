"""Sharded product sumcheck across G devices — orchestration only.

Each round the library computes this rank's partial evaluations (zk_sc_shard_partial), the ranks
all-gather them, and the library adds them and runs the identical transcript step on every rank
(zk_sc_shard_finish).  The production path keeps the exchange inside the library: attach_nccl gives the
context its own NCCL communicator (zk_ctx_attach_nccl, the id broadcast through torch.distributed) and
prove_nccl runs every round with the all-gathers on the context stream (zk_sc_shard_prove_nccl: no
per-round Python, no host synchronisation).  Below `switch_log` local entries the folded tables are all-gathered and the
remaining rounds run on every rank (zk_sc_shard_export / zk_sc_shard_adopt).  The exchange is
behind a tiny `Comm` interface so the same driver runs over NCCL (one process per GPU), gloo (CPU
tests of the host logic with a mock backend) or sequential virtual shards on one device.
"""
from __future__ import annotations

import contextlib
import ctypes

import torch

from . import api
from ._lib import ProdStmt, lib


class ShardSession:
    """zk_sc_shard: this rank's slice of a product-sumcheck statement."""

    def __init__(self, ctx: api.Context, tr: api.Transcript, m: int, n_eq: int, local_tables: list, w: list,
                 rank: int, world: int, claim: int | None = None):
        self.ctx, self.tr, self.m, self.K = ctx, tr, m, len(local_tables)
        self.rank, self.world = rank, world
        mask = 0
        self._ptrs = (ctypes.c_void_p * self.K)()
        self._keep = list(local_tables)
        for k, t in enumerate(local_tables):
            if t.dtype == torch.int32:
                mask |= 1 << k
            self._ptrs[k] = api._dev_ptr(t)
        self._wbuf = api._fr_buf(w)
        stmt = ProdStmt(m, n_eq, self.K, mask, ctypes.cast(self._wbuf, ctypes.c_void_p))
        h = ctypes.c_void_p()
        cb = api._fr_buf([claim]) if claim is not None else None
        ctx.check(lib().zk_sc_shard_create(ctx.h, tr.h, ctypes.byref(stmt), self._ptrs, cb, rank, world, ctypes.byref(h)))
        self.h = h
        self.device = local_tables[0].device
        self.done = False

    @property
    def rounds_done(self) -> int:
        return int(lib().zk_sc_shard_rounds_done(self.h))

    @property
    def local_log(self) -> int:
        return int(lib().zk_sc_shard_local_log(self.h))

    def partial(self) -> torch.Tensor:
        out = torch.empty((self.K + 1, 32), dtype=torch.uint8, device=self.device)
        self.ctx.check(lib().zk_sc_shard_partial(self.h, out.data_ptr()))
        return out

    def finish(self, all_parts: torch.Tensor):
        self.ctx.check(lib().zk_sc_shard_finish(self.h, api._dev_ptr(all_parts)))
        if self.rounds_done == self.m:
            self.done = True

    def export(self) -> torch.Tensor:
        n = 1 << self.local_log
        out = torch.empty((self.K * n, 32), dtype=torch.uint8, device=self.device)
        self.ctx.check(lib().zk_sc_shard_export(self.h, out.data_ptr()))
        return out

    def adopt(self, full: torch.Tensor):
        self.ctx.check(lib().zk_sc_shard_adopt(self.h, api._dev_ptr(full)))
        self.done = True

    def result(self) -> dict:
        plen = ctypes.c_uint64(12 + 32 + 32 * self.m * (self.K + 1) + 32 * self.K)
        proof = ctypes.create_string_buffer(plen.value)
        point = ctypes.create_string_buffer(32 * self.m)
        self.ctx.check(lib().zk_sc_shard_result(self.h, proof, ctypes.byref(plen), point, None, None))
        res = api.parse_sumcheck_proof(proof.raw[:plen.value])
        res["r"] = api._ints(point, self.m)
        res["proof"] = proof.raw[:plen.value]
        return res

    def close(self):
        if getattr(self, "h", None):
            lib().zk_sc_shard_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TorchComm:
    """All-gather over a torch.distributed process group (NCCL on B200s; the buffers stay on device)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        if self.dist.get_backend(self.group) == "nccl":
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        # gloo (tests, CPU hosts of the multi-rank logic): exchange through host memory
        src = t.contiguous().cpu()
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype)
        self.dist.all_gather(list(out.unbind(0)), src, group=self.group)
        return out.to(t.device)


def prove(session, comm, switch_log: int = 12) -> dict:
    """Run the sharded protocol for one rank; every rank returns the same proof.  The torch collectives
    are issued on the session's context stream (the partials are written there)."""
    m = session.m
    ctx = getattr(session, "ctx", None)  # None: a host-side session (the gloo tests' CPU mock)
    with torch.cuda.stream(ctx.stream) if ctx is not None else contextlib.nullcontext():
        while session.rounds_done < m and session.local_log > switch_log:
            session.finish(comm.allgather(session.partial()))
        if not session.done:
            session.adopt(comm.allgather(session.export()))
    return session.result()


def prove_virtual(sessions: list, switch_log: int = 12) -> list:
    """G shards in lockstep in one process (one device): the all-gather is a concatenation."""
    m = sessions[0].m
    while sessions[0].rounds_done < m and sessions[0].local_log > switch_log:
        allp = torch.stack([s.partial() for s in sessions])
        for s in sessions:
            s.finish(allp)
    if not sessions[0].done:
        full = torch.stack([s.export() for s in sessions])
        for s in sessions:
            s.adopt(full)
    return [s.result() for s in sessions]


def attach_nccl(ctx: api.Context, group=None) -> tuple:
    """Give ctx its own NCCL communicator over the ranks of `group` (collective).  Rank 0 of the group
    creates the id (zk_nccl_unique_id), torch.distributed broadcasts it, every rank attaches."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [None]
    if rank == 0:
        buf = ctypes.create_string_buffer(128)
        ctx.check(lib().zk_nccl_unique_id(buf))
        obj[0] = buf.raw[:128]
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    ctx.check(lib().zk_ctx_attach_nccl(ctx.h, obj[0], rank, world))
    return rank, world


def prove_nccl(session: ShardSession, switch_log: int = 12) -> dict:
    """Every remaining round with the library-owned exchange (the session's context attached)."""
    session.ctx.check(lib().zk_sc_shard_prove_nccl(session.h, switch_log))
    session.done = True
    return session.result()
