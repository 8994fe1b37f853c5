"""Row-sharded powerURV for tall A across the GPUs of one box (BASELINE
config C4: powerURV q=1 on 524288 x 4096 fp64 over 1/2/4/8 B200; SURVEY.md
§8e).  The reference (`power_urv_from_sample`, powerurv.py:41-72) is single
process; this is the B200 build's only multi-GPU path.

One process per GPU (SPMD); rank i owns the row block A_i (m_i x n, m_i >= n)
and a replicated G (n x n).  Per power round (powerurv.py:63-68):

  Yhat_i = A_i V                       local DMMA GEMM
  Vhat   = thin Q of Yhat              TSQR: local chunked Householder QRs,
                                       allgather of the n x n R factors, a
                                       redundant QR of the stacked R's, the
                                       explicit Q rebuilt down the tree
  Y      = sum_i A_i^T Vhat_i          local GEMM + allreduce (NCCL)
  Vq     = hqr_full(Y)                 redundant on every rank (n x n)

Final step (powerurv.py:70-71): Ahat_i = A_i Q(Vq) (compact-WY apply), TSQR
of Ahat, then Householder reconstruction of the explicit Q (LU of Q - S,
lu.cu) so that Uq = (Y, Twy) and R match hqr_full(Ahat) up to roundoff.

Only Vhat's column space matters for the next hqr_full (Householder vectors
are invariant under column-sign flips of the input), so the
inner thin QR needs no reconstruction.

PRODUCT PATH: `power_urv_sharded_native` — ONE C-ABI call per rank
(utv_powerurv_sharded_f64, csrc/tsqr.cu) with the collectives inside
libutvb200 on the caller's stream (`NativeComm`: NCCL bootstrapped through
torch.distributed, or an in-process local group of P threads for
single-GPU emulation).

`power_urv_sharded` below is the same SPMD schedule written in Python
against two small interfaces — `Comm` (allreduce / allgather / broadcast)
and an `ops` object — the host-side mirror of tsqr.cu.  It lets the
multi-rank logic run on CPU under torch.distributed/gloo with the numpy
test backend (tests/numpy_ops.py) and on one B200 with `ThreadComm`
(P ranks as threads), so the schedule is validated where no 8-GPU box is
available.
"""

from __future__ import annotations

import threading

from . import device as dv
from ._lib import DMat, dempty


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------

class Comm:
    rank = 0
    size = 1

    def allreduce_sum_(self, t):
        return t

    def allgather(self, t):
        return [t]

    def broadcast_(self, t, src=0):
        return t

    def sync(self):
        """Make this rank's queued device work visible to the collectives."""


class TorchComm(Comm):
    """torch.distributed process group (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce_sum_(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def allgather(self, t):
        out = [t.new_empty(t.shape) for _ in range(self.size)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out

    def broadcast_(self, t, src=0):
        self.dist.broadcast(t, src, group=self.group)
        return t


class _ThreadHub:
    def __init__(self, size):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size


class ThreadComm(Comm):
    """P emulated ranks = P threads of one process on one device.  Each
    thread runs on its own CUDA stream; reductions sum in rank order
    (deterministic)."""

    def __init__(self, hub, rank, stream=None):
        self.hub = hub
        self.rank = rank
        self.size = hub.size
        self.stream = stream

    @staticmethod
    def make(size):
        return _ThreadHub(size)

    def sync(self):
        if self.stream is not None:
            self.stream.synchronize()

    def _exchange(self, t):
        self.sync()
        self.hub.slots[self.rank] = t
        self.hub.barrier.wait()
        return list(self.hub.slots)

    def allreduce_sum_(self, t):
        parts = self._exchange(t)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        self.sync()
        self.hub.barrier.wait()   # everyone has read every slot
        t.copy_(acc)
        self.sync()
        return t

    def allgather(self, t):
        parts = self._exchange(t)
        out = [p.clone() for p in parts]
        self.sync()
        self.hub.barrier.wait()
        return out

    def broadcast_(self, t, src=0):
        parts = self._exchange(t)
        if self.rank != src:
            t.copy_(parts[src])
        self.sync()
        self.hub.barrier.wait()
        return t


# ---------------------------------------------------------------------------
# device building blocks (libutvb200 through device.py)
# ---------------------------------------------------------------------------

class DeviceOps:
    """The building blocks the sharded algorithm needs, on DMat (HBM)."""

    def rows_max(self):
        return dv.geqrf_rows_max()

    def empty(self, rows, cols):
        return dempty(rows, cols)

    def zeros(self, rows, cols):
        m = dempty(rows, cols)
        dv.laset("A", 0.0, 0.0, m)
        return m

    def eye(self, n):
        m = dempty(n, n)
        dv.laset("A", 0.0, 1.0, m)
        return m

    def sub(self, m, r0, c0, nr, nc):
        return m.sub(r0, c0, nr, nc)

    def shape(self, m):
        return m.rows, m.cols

    def copy(self, m):
        return dv.copy(m)

    def lacpy(self, a, b):
        return dv.lacpy(a, b)

    def gemm(self, ta, tb, alpha, a, b, beta=0.0, c=None):
        return dv.gemm(ta, tb, alpha, a, b, beta, c)

    def geqrf(self, a):
        return dv.geqrf(a)

    def larfb(self, side, trans, y, t, b):
        return dv.larfb(side, trans, y, t, b)

    def orgqr(self, y, t, ncols):
        return dv.orgqr(y, t, ncols)

    def getrf_signed(self, a):
        return dv.getrf_signed(a)

    def trsm_right(self, uplo, trans, diag, a, b):
        return dv.trsm_right(uplo, trans, diag, a, b)

    def laset(self, uplo, alpha, beta, a):
        return dv.laset(uplo, alpha, beta, a)

    def tri_zero(self, uplo, a):
        return dv.tri_zero(uplo, a)

    def diag_scale(self, side, d, a, alpha=1.0):
        return dv.diag_scale(side, d, a, alpha)

    # communication payloads: a dense (cols, ld) tensor and back
    def to_comm(self, m):
        if m.off != 0 or m.t.shape[0] != m.cols:
            m = dv.copy(m)
        return m.t

    def from_comm(self, t, rows, cols):
        return DMat(t, rows, cols, t.shape[1])


# ---------------------------------------------------------------------------
# the algorithm
# ---------------------------------------------------------------------------

def _row_chunks(m, n, cap):
    """Split m rows into chunks of <= cap rows, each >= n rows."""
    if m <= cap:
        return [(0, m)]
    k = -(-m // cap)
    base = m // k
    if base < n:
        raise ValueError(f"cannot split {m} rows into chunks of {n}..{cap} rows")
    out, r = [], 0
    for i in range(k):
        nr = base + (1 if i < m % k else 0)
        out.append((r, nr))
        r += nr
    return out


def tsqr(x, comm, ops, chunk_rows=None):
    """Distributed thin QR of the row-sharded x (this rank: m_i x n, m_i >= n).

    Returns (Q_i explicit m_i x n, R n x n replicated, upper with zeros below).
    Tree: local row chunks -> stacked local R's -> allgather -> stacked
    global R's; Q is rebuilt top-down by compact-WY applications."""
    m, n = ops.shape(x)
    if m < n:
        raise ValueError(f"every rank needs at least n = {n} rows, rank {comm.rank} has {m}")
    cap = min(chunk_rows or ops.rows_max(), ops.rows_max())
    chunks = _row_chunks(m, n, cap)
    work = ops.copy(x)
    leaves = []
    for (r0, nr) in chunks:
        blk = ops.sub(work, r0, 0, nr, n)
        y, t = ops.geqrf(blk)                    # blk <- R_c (zeros below)
        leaves.append((y, t))
    nch = len(chunks)
    if nch > 1:
        stk = ops.empty(nch * n, n)
        for c, (r0, _) in enumerate(chunks):
            ops.lacpy(ops.sub(work, r0, 0, n, n), ops.sub(stk, c * n, 0, n, n))
        ys, ts = ops.geqrf(stk)
        r_loc = ops.sub(stk, 0, 0, n, n)
    else:
        ys = ts = None
        r_loc = ops.sub(work, 0, 0, n, n)
    # ---- across ranks ----
    if comm.size > 1:
        comm.sync()
        parts = comm.allgather(ops.to_comm(ops.copy(r_loc)))
        gst = ops.empty(comm.size * n, n)
        for p, tp in enumerate(parts):
            ops.lacpy(ops.from_comm(tp, n, n), ops.sub(gst, p * n, 0, n, n))
        yg, tg = ops.geqrf(gst)                  # redundant on every rank (same bits)
        r = ops.copy(ops.sub(gst, 0, 0, n, n))
        e = ops.orgqr(yg, tg, n)                 # (P n) x n
        e_i = ops.sub(e, comm.rank * n, 0, n, n)
    else:
        r = ops.copy(r_loc)
        e_i = ops.eye(n)
    # ---- back down the local tree ----
    if nch > 1:
        f = ops.empty(nch * n, n)
        q_times_top(ys, ts, e_i, f, ops)
        tops = [ops.sub(f, c * n, 0, n, n) for c in range(nch)]
    else:
        tops = [e_i]
    q = ops.empty(m, n)
    for c, (r0, nr) in enumerate(chunks):
        y, t = leaves[c]
        q_times_top(y, t, tops[c], ops.sub(q, r0, 0, nr, n), ops)
    return q, r


def q_times_top(y, t, top, out, ops):
    """out = Q [top; 0] for Q = I - Y T Y^T (y: k x n unit lower, t: the full
    n x n forward triangle, top: n x n).  The zero block below top is never
    touched: W = T (Y1^T top) costs 2 n^3 each, then out = [top; 0] - Y W is
    one k x n x n product — half the flops of a dense larfb on [top; 0]."""
    k, n = ops.shape(y)
    y1 = ops.sub(y, 0, 0, n, n)
    w = ops.gemm("N", "N", 1.0, t, ops.gemm("T", "N", 1.0, y1, top))
    o1 = ops.sub(out, 0, 0, n, n)
    ops.lacpy(top, o1)
    ops.gemm("N", "N", -1.0, y1, w, 1.0, o1)
    if k > n:
        ops.gemm("N", "N", -1.0, ops.sub(y, n, 0, k - n, n), w, 0.0, ops.sub(out, n, 0, k - n, n))
    return out


def householder_from_q(q, r_in, comm, ops):
    """Compact-WY factor (Y_i rows, Twy) and R of hqr_full for the sharded
    explicit thin Q (LAPACK dorhr_col; lu.cu).  Rank 0 must own >= n rows.

    Only the top n x n block is factored (on rank 0): Q_0[:n] - S = L11 U'.
    It is broadcast with S, and every rank then forms its own rows of
    Y = Q U'^{-1} by a triangular solve (the rows below the top block are
    unshifted, so L21 = Q21 U'^{-1}); rank 0's top rows are L11."""
    m, n = ops.shape(q)
    if comm.rank == 0:
        top = ops.copy(ops.sub(q, 0, 0, n, n))
        s = ops.getrf_signed(top)                # top = L11 \ U'
    else:
        top = ops.empty(n, n)
        s = None
    if comm.size > 1:
        comm.sync()
        ttop = ops.to_comm(top)
        comm.broadcast_(ttop, 0)
        top = ops.from_comm(ttop, n, n)
        s = comm.broadcast_(s if s is not None else _vec_like(ttop, n), 0)
    y = q
    if comm.rank == 0:
        y1 = ops.sub(y, 0, 0, n, n)
        ops.lacpy(top, y1)
        ops.laset("U", 0.0, 1.0, y1)                       # unit lower L11 on top
        if m > n:
            ops.trsm_right("U", "N", "N", top, ops.sub(y, n, 0, m - n, n))
    else:
        ops.trsm_right("U", "N", "N", top, y)              # Y_i = Q_i U'^{-1}
    # Twy = -U' S L11^{-T}, redundantly on every rank
    tw = ops.copy(top)
    ops.tri_zero("L", tw)                                  # U' (upper incl. diagonal)
    ops.diag_scale("R", s, tw, -1.0)                       # -U' S
    ops.trsm_right("L", "T", "U", top, tw)                 # ... L11^{-T}
    # R = S R_tsqr
    r = ops.copy(r_in)
    ops.diag_scale("L", s, r, 1.0)
    return y, tw, r, s


def _vec_like(t, n):
    return t.new_empty(n)


def power_urv_sharded(a_loc, g, q, comm=None, ops=None, chunk_rows=None):
    """Row-sharded powerURV (power_urv_from_sample, powerurv.py:41-72) — SPMD.

    a_loc: this rank's row block of A (m_i x n); g: the replicated n x n
    Gaussian G.  Returns dict with this rank's rows of Uq.Y (Uy), and the
    replicated Uq.Twy (Ut), R (n x n; rows n.. of the reference's m x n R are
    zero), Vq.Y (Vy) and Vq.Twy (Vt)."""
    comm = comm or Comm()
    ops = ops or DeviceOps()
    m, n = ops.shape(a_loc)
    if q < 0:
        raise ValueError(f"power iteration count must be >= 0, got {q}")
    if q == 0:
        vy, vt = ops.geqrf(ops.copy(g))              # powerurv.py:58-59
    else:
        v = g
        for it in range(q):                          # powerurv.py:63-68
            yhat = ops.gemm("N", "N", 1.0, a_loc, v)                 # :64
            vhat, _ = tsqr(yhat, comm, ops, chunk_rows)              # :65
            del yhat
            y = ops.gemm("T", "N", 1.0, a_loc, vhat)                 # :66 (partial)
            del vhat
            if comm.size > 1:
                comm.sync()
                ty = ops.to_comm(y)
                comm.allreduce_sum_(ty)
                y = ops.from_comm(ty, n, n)
            vy, vt = ops.geqrf(y)                                    # :67
            if it + 1 < q:
                v = ops.orgqr(vy, vt, n)                             # :68
    # :70 A Q(Vq): V explicit (n x n, 2n^3) and one m_i x n x n product, not
    # a compact-WY apply to a copy of A (>= 4 m_i n^2 for n reflectors)
    ahat = ops.gemm("N", "N", 1.0, a_loc, ops.orgqr(vy, vt, n))
    qh, r_in = tsqr(ahat, comm, ops, chunk_rows)                     # :71
    del ahat
    uy, ut, r, _ = householder_from_q(qh, r_in, comm, ops)
    return {"Uy": uy, "Ut": ut, "R": r, "Vy": vy, "Vt": vt}


# ---------------------------------------------------------------------------
# product path: the whole SPMD schedule inside libutvb200 (csrc/tsqr.cu)
# ---------------------------------------------------------------------------

class NativeComm:
    """A libutvb200 communicator (utv_comm_t, csrc/comm.cu)."""

    def __init__(self, handle):
        from ._lib import load
        self._lib = load()
        self.handle = handle
        self.rank = self._lib.utv_comm_rank(handle)
        self.size = self._lib.utv_comm_size(handle)

    @classmethod
    def nccl(cls, group=None):
        """NCCL communicator over the ranks of a torch.distributed group (one
        process per GPU, current device bound); torch.distributed only ships
        the 128-byte unique id from rank 0."""
        import ctypes

        import torch.distributed as dist
        from ._lib import check, load
        lib = load()
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        buf = ctypes.create_string_buffer(128)
        if rank == 0:
            check(lib.utv_comm_nccl_unique_id(buf), "utv_comm_nccl_unique_id")
        obj = [buf.raw if rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(obj, src=src, group=group)
        uid = ctypes.create_string_buffer(obj[0], 128)
        h = ctypes.c_void_p()
        check(lib.utv_comm_init_nccl(uid, size, rank, ctypes.byref(h)), "utv_comm_init_nccl")
        return cls(h.value)

    @classmethod
    def nccl_single(cls):
        """A 1-rank NCCL communicator (no torch.distributed needed)."""
        import ctypes

        from ._lib import check, load
        lib = load()
        uid = ctypes.create_string_buffer(128)
        check(lib.utv_comm_nccl_unique_id(uid), "utv_comm_nccl_unique_id")
        h = ctypes.c_void_p()
        check(lib.utv_comm_init_nccl(uid, 1, 0, ctypes.byref(h)), "utv_comm_init_nccl")
        return cls(h.value)

    @classmethod
    def local_group(cls, size):
        """`size` in-process ranks (drive each from its own thread + stream)."""
        import ctypes

        from ._lib import check, load
        hs = (ctypes.c_void_p * size)()
        check(load().utv_comm_init_local(size, hs), "utv_comm_init_local")
        return [cls(hs[r]) for r in range(size)]

    def close(self):
        if self.handle:
            self._lib.utv_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass


def power_urv_sharded_native(a_loc, g, q, comm, chunk_rows=None):
    """Row-sharded powerURV (power_urv_from_sample, powerurv.py:41-72): one
    utv_powerurv_sharded_f64 call on this rank.  a_loc: this rank's rows of A
    (DMat, m_i x n, m_i >= n); g: the replicated n x n G (DMat); comm: a
    NativeComm.  Returns dict(Uy = this rank's rows of Uq.Y, Ut, R (n x n),
    Vy, Vt) as DMats.  Every rank must call it (collective); it runs on
    torch's current stream (the workspace is released to the caching
    allocator in that stream's order)."""
    from ._lib import check, dempty, load, stream_ptr, workspace
    lib = load()
    m, n = a_loc.rows, a_loc.cols
    if q < 0:
        raise ValueError(f"power iteration count must be >= 0, got {q}")
    cr = int(chunk_rows or 0)
    out = {"Uy": dempty(m, n), "Ut": dempty(n, n), "R": dempty(n, n), "Vy": dempty(n, n),
           "Vt": dempty(n, n)}
    lw = lib.utv_powerurv_sharded_bufsize(m, n, comm.size, cr)
    ws = workspace(lw)
    st = stream_ptr()
    check(lib.utv_powerurv_sharded_f64(
        comm.handle, m, n, int(q), a_loc.ptr, a_loc.ld, g.ptr, g.ld,
        out["Uy"].ptr, out["Uy"].ld, out["Ut"].ptr, out["Ut"].ld, out["R"].ptr, out["R"].ld,
        out["Vy"].ptr, out["Vy"].ld, out["Vt"].ptr, out["Vt"].ld, cr, ws.data_ptr(), lw, st),
        "utv_powerurv_sharded_f64")
    return out
