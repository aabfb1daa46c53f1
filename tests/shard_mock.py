"""CPU stand-in for paper_2307_16273_b200.shard.ShardSession (test infrastructure).

Same methods, plain Python integers, the definitions of Protocol 3's round messages
restricted to this rank's slice.  It lets the sharding host logic (slicing on the high index bits,
the rank eq factor, round-by-round all-gather + identical transcript steps, the gather switch and
continuation) run under torch.distributed/gloo on CPU, where the CUDA kernels cannot.
"""
import torch

P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def _eq(u, bits_value, n):
    e = 1
    for t in range(n):
        e = e * (u[t] if (bits_value >> t) & 1 else 1 - u[t]) % P
    return e


def _enc(vals):
    return torch.frombuffer(bytearray(b"".join(int(v).to_bytes(32, "little") for v in vals)), dtype=torch.uint8).reshape(-1, 32)


def _dec(t):
    raw = t.contiguous().numpy().tobytes()
    return [int.from_bytes(raw[32 * i:32 * i + 32], "little") for i in range(len(raw) // 32)]


class MockSession:
    def __init__(self, tr, m, n_eq, local_tables, w, rank, world, claim=None):
        self.tr, self.m, self.n_eq, self.K, self.w = tr, m, n_eq, len(local_tables), list(w)
        self.rank, self.world = rank, world
        s = world.bit_length() - 1
        self.L = m - s
        self.T = [[v % P for v in t] for t in local_tables]
        self.t = 0
        self.t0 = 0
        self.claim_given = claim is not None
        self.claim = claim
        self.msgs = []
        self.r = []
        self.done = False
        hdr = b"".join(int(x).to_bytes(4, "little") for x in (m, n_eq, self.K))
        tr.absorb("sc/hdr", hdr)
        if self.claim_given:
            tr.absorb("sc/claim", int(claim).to_bytes(32, "little"))
        # rank eq factor over the high bits that the eq covers
        self.scale = _eq(self.w[self.L:], rank, n_eq - self.L) if n_eq > self.L else 1
        self.n_eq_loc = min(n_eq, self.L)

    @property
    def rounds_done(self):
        return self.t

    @property
    def local_log(self):
        return len(self.T[0]).bit_length() - 1

    def _message(self, T, t, n_eq_end):
        half = len(T[0]) // 2
        ev = []
        for X in range(self.K + 1):
            acc = 0
            for b in range(half):
                e = 1
                if t < n_eq_end:
                    nv = n_eq_end - t - 1
                    e = _eq(self.w[t + 1:], b & ((1 << nv) - 1), nv)
                p = e
                for tb in T:
                    p = p * (tb[2 * b] + X * (tb[2 * b + 1] - tb[2 * b])) % P
                acc += p
            ev.append(acc % P)
        return ev

    def partial(self):
        ev = self._message(self.T, self.t, self.n_eq_loc)
        self.t += 1
        return _enc([v * self.scale % P for v in ev])

    def _step(self, ev):
        t = len(self.msgs)
        if t == 0 and not self.claim_given:
            if t < self.n_eq:
                self.claim = ((1 - self.w[0]) * ev[0] + self.w[0] * ev[1]) % P
            else:
                self.claim = (ev[0] + ev[1]) % P
            self.tr.absorb("sc/claim", self.claim.to_bytes(32, "little"))
        self.tr.absorb("sc/msg", b"".join(v.to_bytes(32, "little") for v in ev))
        r = self.tr.challenges("sc/r", 1)[0]
        self.msgs.append(ev)
        self.r.append(r)
        self.T = [[(tb[2 * b] + r * (tb[2 * b + 1] - tb[2 * b])) % P for b in range(len(tb) // 2)] for tb in self.T]
        return r

    def finish(self, all_parts):
        allv = _dec(all_parts.reshape(-1, 32))
        K1 = self.K + 1
        ev = [sum(allv[g * K1 + x] for g in range(self.world)) % P for x in range(K1)]
        self._step(ev)
        if self.t == self.m:
            self._finals()

    def export(self):
        return _enc([v for tb in self.T for v in tb])

    def adopt(self, full):
        allv = _dec(full.reshape(-1, 32))
        n = len(self.T[0])
        self.T = [[allv[(g * self.K + k) * n + j] for g in range(self.world) for j in range(n)] for k in range(self.K)]
        while self.t < self.m:
            ev = self._message(self.T, self.t, self.n_eq)     # full tables: eq over w[t+1 .. n_eq-1]
            self.t += 1
            self._step(ev)
        self._finals()

    def _finals(self):
        fin = [tb[0] for tb in self.T]
        self.tr.absorb("sc/final", b"".join(v.to_bytes(32, "little") for v in fin))
        self.finals = fin
        self.done = True

    def result(self):
        return dict(claim=self.claim, msgs=self.msgs, r=self.r, finals=self.finals, state=self.tr.state())
