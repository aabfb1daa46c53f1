"""Quantized FCN training trace and FAC4DNN family assembly (input generation only).

The prover's input is the training trace of PAPER.md Example 2 (L292-312):
    Z^(l)   = A^(l-1) W^(l)                              (Eq. fcnn-Z)
    A^(l)   = ReLU(round(Z^(l) / 2^R)),  1 <= l <= L-1    (L170)
    G_Z^(L) = round(Z^(L) / 2^R) - Y                      (Eq. fcnn-GZ-last, rescaled once: DESIGN.md D16)
    G_A^(l) = G_Z^(l+1) W^(l+1)^T,       1 <= l <= L-1    (Eq. fcnn-GA)
    G_Z^(l) = 1{Z^(l) >= 0} * round(G_A^(l) / 2^R)        (L177, Lemma 1)
    G_W^(l) = G_Z^(l)^T A^(l-1),         1 <= l <= L      (Eq. fcnn-GW)
    W^(l)  -= round(G_W^(l)^T / 2^20)                     (optimizer unspecified, L309; trace only)
round() is half-up (D9).  This module runs the *training* (the
prover's input, Protocol 1 line 2), never any part of the proof.  Matmuls run
in float64 BLAS, exact because every partial sum is an integer below 2^53
(|entries| < 2^13, inner dimension <= 4096).

Families: every forward / input-gradient /
weight-gradient matmul and every ReLU is grouped by (equation type, shape);
instances are ordered by (step, layer) and the stack axis is zero-padded to a
power of two.  The family order is fixed: ReLU families, then all
F, then GA, then GW families (each in increasing first-layer order).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .prng import DATA_SEED, uniform_range

R_BITS = 16
Q_BITS = 16
LR_SHIFT = 20


def _round_half_up(x: np.ndarray, r: int) -> np.ndarray:
    return (x + (1 << (r - 1))) >> r


def _matmul_exact(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    out = (a.astype(np.float64) @ b.astype(np.float64))
    res = np.rint(out).astype(np.int64)
    return res


def _to_i32(x: np.ndarray, what: str) -> np.ndarray:
    lim = 1 << 31
    if x.size and (x.max() >= lim or x.min() < -lim):
        raise OverflowError(f"{what} leaves int32: [{x.min()}, {x.max()}]")
    return x.astype(np.int32)


@dataclass
class FcnShape:
    name: str
    dims: list            # padded widths d_0 .. d_L (powers of two)
    real_dims: list       # unpadded widths
    batch: int
    steps: int            # T'


C3_SHAPE = FcnShape("C3", [1024] * 9, [1024] * 9, 64, 1)
C4_SHAPE = FcnShape("C4", [4096] + [1024] * 8 + [16], [3072] + [1024] * 8 + [10], 64, 16)


def tiny_shape(steps=2, layers=3, width=8, batch=4, din=8, dout=4):
    dims = [din] + [width] * (layers - 1) + [dout]
    return FcnShape(f"tiny{layers}x{width}", dims, list(dims), batch, steps)


@dataclass
class StepTrace:
    A: list = field(default_factory=list)    # A[0] = X, A[l] for l=1..L-1 (int32 [B, d_l])
    Z: list = field(default_factory=list)    # Z[l] for l=1..L (index 0 unused)
    W: list = field(default_factory=list)    # W[l] [d_{l-1}, d_l] for l=1..L
    GZ: list = field(default_factory=list)   # G_Z[l] for l=1..L
    GA: list = field(default_factory=list)   # G_A[l] for l=1..L-1
    GW: list = field(default_factory=list)   # G_W[l] [d_l, d_{l-1}] for l=1..L
    Zp: np.ndarray = None                     # round(Z^(L) / 2^R) (D16) [B, d_L]
    Y: np.ndarray = None                      # labels: Zp - G_Z^(L) [B, d_L]


def _pad_mask(shape: FcnShape, l: int):
    """Boolean mask of the real (unpadded) entries of W^(l)."""
    r_in, r_out = shape.real_dims[l - 1], shape.real_dims[l]
    m = np.zeros((shape.dims[l - 1], shape.dims[l]), dtype=bool)
    m[:r_in, :r_out] = True
    return m


def generate_trace(shape: FcnShape, seed: int = DATA_SEED, x_bits=11, w_bits=12, y_bits=10):
    """Run T' quantized SGD steps; returns a list of StepTrace (one per step)."""
    L = len(shape.dims) - 1
    B = shape.batch
    W = [None]
    for l in range(1, L + 1):
        w = uniform_range(seed, 1000 + l, (shape.dims[l - 1], shape.dims[l]), -(1 << w_bits), 1 << w_bits).astype(np.int64)
        w[~_pad_mask(shape, l)] = 0
        W.append(w)
    steps = []
    for s in range(shape.steps):
        tr = StepTrace()
        x = uniform_range(seed, 100000 + s, (B, shape.dims[0]), -(1 << x_bits), 1 << x_bits).astype(np.int64)
        x[:, shape.real_dims[0]:] = 0
        A = [x]
        Z = [None]
        for l in range(1, L + 1):
            z = _matmul_exact(A[l - 1], W[l])
            _to_i32(z, f"Z^{l}")
            Z.append(z)
            if l < L:
                A.append(np.where(z >= 0, _round_half_up(z, R_BITS), 0))
        noise = uniform_range(seed, 200000 + s, (B, shape.dims[L]), -(1 << y_bits), 1 << y_bits).astype(np.int64)
        noise[:, shape.real_dims[L]:] = 0
        GZ = [None] * (L + 1)
        GA = [None] * (L + 1)
        GZ[L] = noise                     # = round(Z^(L)/2^R) - Y with Y := round(Z^(L)/2^R) - noise
        for l in range(L - 1, 0, -1):
            ga = _matmul_exact(GZ[l + 1], W[l + 1].T)
            _to_i32(ga, f"G_A^{l}")
            GA[l] = ga
            GZ[l] = np.where(Z[l] >= 0, _round_half_up(ga, R_BITS), 0)
        GW = [None]
        for l in range(1, L + 1):
            gw = _matmul_exact(GZ[l].T, A[l - 1])
            _to_i32(gw, f"G_W^{l}")
            GW.append(gw)
        tr.A = [_to_i32(a, "A") for a in A]
        tr.Z = [None] + [_to_i32(z, "Z") for z in Z[1:]]
        tr.W = [None] + [_to_i32(w, "W") for w in W[1:]]
        tr.GZ = [None] + [_to_i32(g, "G_Z") for g in GZ[1:]]
        tr.GA = [None] + [_to_i32(GA[l], "G_A") for l in range(1, L)]
        tr.GW = [None] + [_to_i32(g, "G_W") for g in GW[1:]]
        tr.Zp = _to_i32(_round_half_up(Z[L], R_BITS), "Z'^L")
        tr.Y = _to_i32(tr.Zp.astype(np.int64) - GZ[L], "Y")
        steps.append(tr)
        for l in range(1, L + 1):
            W[l] = W[l] - _round_half_up(GW[l].T.astype(np.int64), LR_SHIFT)
            W[l][~_pad_mask(shape, l)] = 0
    return steps


def _next_pow2(n: int) -> int:
    return 1 << max(0, (n - 1).bit_length())


def _stack(mats, n_pad):
    shp = mats[0].shape
    out = np.zeros((n_pad,) + shp, dtype=np.int32)
    for i, m in enumerate(mats):
        out[i] = m
    return out


@dataclass
class MatmulFamily:
    """Y[n] = op(A[n]) @ op(B[n]) for n < N (zero instances beyond the real count).

    A is stored [N][D1][D2] (transA=False) or [N][D2][D1] (transA=True);
    B is stored [N][D2][D3] (transB=False) or [N][D3][D2] (transB=True).
    Y ([N][D1][D3]) is the trace's product tensor, kept for the oracle's checks.
    """
    name: str
    A: np.ndarray
    B: np.ndarray
    Y: np.ndarray
    transA: bool
    transB: bool
    n_real: int
    insts: list = field(default_factory=list)   # (step, layer) per stack slot
    refs: dict = field(default_factory=dict)    # plan_window: role "A" / "B" / "Y" -> TensorRef

    @property
    def logs(self):
        N = self.A.shape[0]
        D1 = self.A.shape[2] if self.transA else self.A.shape[1]
        D2 = self.A.shape[1] if self.transA else self.A.shape[2]
        D3 = self.B.shape[1] if self.transB else self.B.shape[2]
        return tuple(int(v).bit_length() - 1 for v in (N, D1, D2, D3))


@dataclass
class ReluFamily:
    """Stacked zkReLU instances: Z, G_A flattened to [D] int32 (D = N * per-instance size)."""
    name: str
    Z: np.ndarray
    GA: np.ndarray
    Q: int
    R: int
    n_real: int
    insts: list = field(default_factory=list)
    tensors: dict = field(default_factory=dict)  # plan_window: "Z" / "A" / "GA" / "GZ" -> tensor family name


def assemble_families(shape: FcnShape, trace):
    """Group the trace's operations into FAC4DNN families (fixed order, see module doc)."""
    L = len(shape.dims) - 1
    fam = []
    cache = {}

    def stk(field, idx, N):
        # one array per distinct stack: e.g. W[2..8] is the B operand of F[2..8] and of GA[1..7],
        # A[1..7] of F[2..8] and GW[2..8], G_Z[2..8] of GA[1..7] and GW[2..8]
        key = (field, tuple(idx), N)
        if key not in cache:
            cache[key] = _stack([getattr(trace[s], field)[l] for s, l in idx], N)
        return cache[key]

    def group(kind, layers, key_fn):
        groups = {}
        for l in layers:
            groups.setdefault(key_fn(l), []).append(l)
        return sorted(groups.items(), key=lambda kv: kv[1][0])

    # zkReLU after every hidden layer (first: the most proving work on the least data, so an
    # end-to-end prover's uploads of the large matmul stacks overlap it)
    for key, ls in group("ReLU", range(1, L), lambda l: shape.dims[l]):
        insts = [(s, l) for s in range(shape.steps) for l in ls]
        N = _next_pow2(len(insts))
        per = shape.batch * shape.dims[ls[0]]
        Z = np.zeros(N * per, dtype=np.int32)
        G = np.zeros(N * per, dtype=np.int32)
        for i, (s, l) in enumerate(insts):
            Z[i * per:(i + 1) * per] = trace[s].Z[l].reshape(-1)
            G[i * per:(i + 1) * per] = trace[s].GA[l].reshape(-1)
        fam.append(ReluFamily(f"ReLU[{','.join(map(str, ls))}]", Z, G, Q_BITS, R_BITS, len(insts), insts))
    # forward: Z^(l) = A^(l-1) W^(l).  The key also separates the first layer (its input is the data X)
    # and the top layer (its output is not ReLU'd), so every operand stack of a family is a view of ONE
    # tensor family (plan_window)
    for key, ls in group("F", range(1, L + 1), lambda l: (shape.dims[l - 1], shape.dims[l], l == 1, l == L)):
        insts = [(s, l) for s in range(shape.steps) for l in ls]
        N = _next_pow2(len(insts))
        fam.append(MatmulFamily(
            f"F[{','.join(map(str, ls))}]",
            stk("A", [(s, l - 1) for s, l in insts], N),
            stk("W", [(s, l) for s, l in insts], N),
            stk("Z", [(s, l) for s, l in insts], N), False, False, len(insts), insts))
    # input gradients: G_A^(l) = G_Z^(l+1) W^(l+1)^T
    for key, ls in group("GA", range(1, L), lambda l: (shape.dims[l + 1], shape.dims[l], l + 1 == L)):
        insts = [(s, l) for s in range(shape.steps) for l in ls]
        N = _next_pow2(len(insts))
        fam.append(MatmulFamily(
            f"GA[{','.join(map(str, ls))}]",
            stk("GZ", [(s, l + 1) for s, l in insts], N),
            stk("W", [(s, l + 1) for s, l in insts], N),
            stk("GA", [(s, l) for s, l in insts], N), False, True, len(insts), insts))
    # weight gradients: G_W^(l) = G_Z^(l)^T A^(l-1)
    for key, ls in group("GW", range(1, L + 1), lambda l: (shape.dims[l], shape.dims[l - 1], l == 1, l == L)):
        insts = [(s, l) for s in range(shape.steps) for l in ls]
        N = _next_pow2(len(insts))
        fam.append(MatmulFamily(
            f"GW[{','.join(map(str, ls))}]",
            stk("GZ", [(s, l) for s, l in insts], N),
            stk("A", [(s, l - 1) for s, l in insts], N),
            stk("GW", [(s, l) for s, l in insts], N), True, False, len(insts), insts))
    return fam


@dataclass
class LossFamily:
    """Eq. (fcnn-GZ-last) at the activations' scale (D16): G_Z^(L) = Z^(L)' - Y, stacked over the
    window's steps (D24); GZ, Zp, Y: [N][B][d_L]."""
    name: str
    GZ: np.ndarray
    Zp: np.ndarray
    Y: np.ndarray
    insts: list = field(default_factory=list)
    refs: dict = field(default_factory=dict)    # plan_window: "GZ" / "Zp" / "Y" -> TensorRef


@dataclass
class RescaleFamily:
    """The top layer's Z^(L) = 2^R Z^(L)' + R_Z, proved through the bits of Z^(L) (D26);
    Z: the stacked Z^(L) flattened, [N * B * d_L]."""
    name: str
    Z: np.ndarray
    Q: int
    R: int
    insts: list = field(default_factory=list)
    tensors: dict = field(default_factory=dict)  # plan_window: "Z" -> "Zout", "Zp" -> "Zp"


def assemble_top_families(shape: FcnShape, trace, families: list) -> list:
    """The loss-gradient and rescale families of the top layer (N2), stacked over the steps like every
    family; the G_Z^(L) stack is the one the GA family of the top layer already holds."""
    L = len(shape.dims) - 1
    insts = [(s, L) for s in range(shape.steps)]
    N = _next_pow2(len(insts))
    ga_top = next((f for f in families if f.name.startswith("GA[") and max(l for _, l in f.insts) == L - 1), None)
    gz = ga_top.A if ga_top is not None and ga_top.A.shape[0] == N else _stack([trace[s].GZ[L] for s, _ in insts], N)
    zp = _stack([trace[s].Zp for s, _ in insts], N)
    y = _stack([trace[s].Y for s, _ in insts], N)
    f_top = next((f for f in families if f.name.startswith("F[") and max(l for _, l in f.insts) == L), None)
    z = f_top.Y if f_top is not None and f_top.Y.shape[0] == N else _stack([trace[s].Z[L] for s, _ in insts], N)
    return [LossFamily(f"Loss[{L}]", gz, zp, y, insts), RescaleFamily(f"Rescale[{L}]", z.reshape(-1), Q_BITS, R_BITS, insts)]


def fcn_header(shape: FcnShape) -> bytes:
    """Bytes absorbed under tag "fcn/hdr" before the first family (D3d)."""
    words = [len(shape.dims) - 1, shape.batch, shape.steps] + list(shape.dims)
    return b"".join(int(w).to_bytes(4, "little") for w in words)


# ---------------------------------------------------------------- tensor families (Protocol 1)
@dataclass
class TensorFamily:
    """A stack S_i of same-kind, same-shape tensors of the window (Protocol 1 line 4): slot j holds
    the tensor of (step, layer) slots[j] (None: an all-zero slot), each stored [rows][cols] as the trace
    holds it.  relu: the ReLU family whose aux binds the tensor (Z, A, G_A, G_Z: P:L274) — its values are
    then formed from that family's Z / G_A words — else None (a committed tensor, array = its stack)."""
    name: str
    kind: str
    slots: list
    rows: int
    cols: int
    relu: str | None = None
    array: np.ndarray | None = None


@dataclass
class TensorRef:
    """A family operand as a view of a tensor family: family slot n holds tensor slot map[n] (-1: zero)."""
    tensor: str
    map: list


# (field, layer) -> tensor-family kind
def _kind(field_: str, l: int, L: int) -> str:
    if field_ == "A":
        return "X" if l == 0 else "A"
    if field_ in ("Z", "GZ"):
        return field_ + ("out" if l == L else "")
    return field_                      # GA (hidden only), W, GW


def plan_window(shape: FcnShape, trace, families: list, top: list | None = None) -> list:
    """Tensor families of a window and the views the operation families take of them (input structure
    only: which stored tensor each stack slot is).  Sets f.refs (matmul families: roles "A", "B", "Y")
    and f.tensors (ReLU families) and returns the tensor families in a fixed order: X, then per ReLU
    family its Z, A, G_A, G_Z, then Zout, GZout, W and GW groups (in family order)."""
    L = len(shape.dims) - 1
    relus = [f for f in families if isinstance(f, ReluFamily)]
    mms = [f for f in families if hasattr(f, "A")]
    loss = next((f for f in (top or []) if isinstance(f, LossFamily)), None)
    resc = next((f for f in (top or []) if isinstance(f, RescaleFamily)), None)
    tf = {}
    order = []

    def add(name, kind, slots, rows, cols, relu=None, array=None):
        if name not in tf:
            tf[name] = TensorFamily(name, kind, slots, rows, cols, relu, array)
            order.append(name)
        return tf[name]

    def stack(field_, slots, rows, cols):
        out = np.zeros((len(slots), rows, cols), dtype=np.int32)
        for j, sl in enumerate(slots):
            if sl is not None:
                out[j] = getattr(trace[sl[0]], field_)[sl[1]]
        return out

    def pad(slots):
        return slots + [None] * (_next_pow2(len(slots)) - len(slots))

    def same(slots, f, role):    # the family's own operand stack when it holds exactly these slots
        if f is None or len(slots) != getattr(f, role).shape[0]:
            return None
        want = [None] * len(slots)
        for j, (s, l) in enumerate(f.insts):
            want[j] = {"F": {"A": (s, l - 1), "B": (s, l), "Y": (s, l)},
                       "GA": {"A": (s, l + 1), "B": (s, l + 1), "Y": (s, l)},
                       "GW": {"A": (s, l), "B": (s, l - 1), "Y": (s, l)}}[f.name.split("[")[0]][role]
        return getattr(f, role) if want == slots else None

    def first(pred):
        return next((f for f in mms if pred(f)), None)

    B = shape.batch
    xs = pad([(s, 0) for s in range(shape.steps)])
    f1 = first(lambda f: f.name.startswith("F[") and min(l for _, l in f.insts) == 1)
    xa = same(xs, f1, "A")
    add("X", "X", xs, B, shape.dims[0], array=xa if xa is not None else stack("A", xs, B, shape.dims[0]))
    home = {}                     # (kind, layer) -> tensor family name
    for f in relus:
        lay = sorted({l for _, l in f.insts})
        tag = ",".join(map(str, lay))
        slots = pad(list(f.insts))
        w = shape.dims[lay[0]]
        f.tensors = {}
        for k in ("Z", "A", "GA", "GZ"):
            nm = f"{k}[{tag}]"
            add(nm, k, slots, B, w, relu=f.name)
            f.tensors[k] = nm
            for l in lay:
                home[(k, l)] = nm
    zs = pad([(s, L) for s in range(shape.steps)])
    fL = first(lambda f: f.name.startswith("F[") and max(l for _, l in f.insts) == L)
    gL = first(lambda f: f.name.startswith("GA[") and max(l for _, l in f.insts) == L - 1)
    za, ga = same(zs, fL, "Y"), same(zs, gL, "A")
    add("Zout", "Zout", zs, B, shape.dims[L], array=za if za is not None else stack("Z", zs, B, shape.dims[L]),
        relu=resc.name if resc is not None else None)
    add("GZout", "GZout", zs, B, shape.dims[L], array=ga if ga is not None else stack("GZ", zs, B, shape.dims[L]))
    if loss is not None:   # the top layer's rescaled output (bound by the rescale's aux) and the labels
        add("Zp", "Zp", zs, B, shape.dims[L], relu=resc.name if resc is not None else None,
            array=loss.Zp if resc is None else None)
        add("Y", "Y", zs, B, shape.dims[L], array=loss.Y)
        loss.refs = {"GZ": TensorRef("GZout", list(range(len(zs)))), "Zp": TensorRef("Zp", list(range(len(zs)))),
                     "Y": TensorRef("Y", list(range(len(zs))))}
    if resc is not None:
        resc.tensors = {"Z": "Zout", "Zp": "Zp"}
    for f in mms:
        if f.name.startswith("F["):
            ls = sorted({l for _, l in f.insts})
            nm = f"W[{','.join(map(str, ls))}]"
            sl = pad(list(f.insts))
            a = same(sl, f, "B")
            add(nm, "W", sl, shape.dims[ls[0] - 1], shape.dims[ls[0]],
                array=a if a is not None else stack("W", sl, shape.dims[ls[0] - 1], shape.dims[ls[0]]))
            for l in ls:
                home[("W", l)] = nm
    for f in mms:
        if f.name.startswith("GW["):
            ls = sorted({l for _, l in f.insts})
            nm = f"GW[{','.join(map(str, ls))}]"
            sl = pad(list(f.insts))
            a = same(sl, f, "Y")
            add(nm, "GW", sl, shape.dims[ls[0]], shape.dims[ls[0] - 1],
                array=a if a is not None else stack("GW", sl, shape.dims[ls[0]], shape.dims[ls[0] - 1]))
            for l in ls:
                home[("GW", l)] = nm
    home[("X", 0)] = "X"
    home[("Zout", L)] = "Zout"
    home[("GZout", L)] = "GZout"

    def ref(keys, N):
        names = {home[(_kind(fl, l, L), l)] for fl, s, l in keys}
        assert len(names) == 1, f"a family operand spans several tensor families: {names}"
        nm = names.pop()
        where = {sl: j for j, sl in enumerate(tf[nm].slots) if sl is not None}
        mp = [where[(s, l)] for fl, s, l in keys] + [-1] * (N - len(keys))
        return TensorRef(nm, mp)

    for f in mms:
        N = f.A.shape[0]
        if f.name.startswith("F["):
            keys = dict(A=[("A", s, l - 1) for s, l in f.insts], B=[("W", s, l) for s, l in f.insts],
                        Y=[("Z", s, l) for s, l in f.insts])
        elif f.name.startswith("GA["):
            keys = dict(A=[("GZ", s, l + 1) for s, l in f.insts], B=[("W", s, l + 1) for s, l in f.insts],
                        Y=[("GA", s, l) for s, l in f.insts])
        else:
            keys = dict(A=[("GZ", s, l) for s, l in f.insts], B=[("A", s, l - 1) for s, l in f.insts],
                        Y=[("GW", s, l) for s, l in f.insts])
        f.refs = {role: ref(k, N) for role, k in keys.items()}
    return [tf[n] for n in order]
