"""ctypes binding of libutvb200.so (include/utv_b200.h) + device-matrix helpers.

PyTorch is used only for device memory, streams and host<->device copies.
There is no CPU fallback: if the library or a CUDA device is missing every
compute entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
import threading
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libutvb200.so")

_lib = None

c_int, c_long, c_double, c_size_t, c_void_p, c_char = (
    ctypes.c_int, ctypes.c_long, ctypes.c_double, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_char)

# name -> (restype, argtypes)
SIGNATURES = {
    "utv_version": (c_int, []),
    "utv_device_sms": (c_int, []),
    "utv_dgemm_bufsize": (c_size_t, [c_int, c_int, c_int]),
    "utv_dgemm": (c_int, [c_char, c_char, c_int, c_int, c_int, c_double, c_void_p, c_long,
                          c_void_p, c_long, c_double, c_void_p, c_long, c_void_p, c_size_t, c_void_p]),
    "utv_dsumsq_bufsize": (c_size_t, []),
    "utv_dsumsq": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_void_p, c_size_t, c_void_p]),
    "utv_dgeqrf_bufsize": (c_size_t, [c_int, c_int]),
    "utv_dgeqrf": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_long, c_void_p, c_long,
                           c_void_p, c_size_t, c_void_p]),
    "utv_dlarfb_bufsize": (c_size_t, [c_int, c_int, c_int]),
    "utv_dlarfb": (c_int, [c_char, c_char, c_int, c_int, c_int, c_int, c_void_p, c_long, c_void_p,
                           c_long, c_void_p, c_long, c_void_p, c_size_t, c_void_p]),
    "utv_dorgqr_bufsize": (c_size_t, [c_int, c_int, c_int]),
    "utv_dorgqr": (c_int, [c_int, c_int, c_int, c_void_p, c_long, c_void_p, c_long, c_void_p,
                           c_long, c_void_p, c_size_t, c_void_p]),
    "utv_dgesvj_bufsize": (c_size_t, [c_int]),
    "utv_dgesvj": (c_int, [c_int, c_void_p, c_long, c_void_p, c_void_p, c_long, c_void_p, c_long,
                           c_void_p, c_void_p, c_size_t, c_void_p]),
    "utv_dgesvj_ex": (c_int, [c_int, c_void_p, c_long, c_void_p, c_void_p, c_long, c_void_p, c_long,
                              c_void_p, c_int, c_void_p, c_size_t, c_void_p]),
    "utv_randutv_basic_bufsize": (c_size_t, [c_int, c_int, c_int, c_int]),
    "utv_randutv_basic_f64": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_long, c_void_p,
                                      c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "utv_randutv_basic_steps_f64": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                            c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                            c_long, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_size_t, c_void_p]),
    "utv_randutv_basic_steps_carry_f64": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                                                  c_void_p, c_long, c_void_p, c_long, c_void_p, c_long,
                                                  c_void_p, c_long, c_void_p, c_void_p, c_void_p,
                                                  c_void_p, c_size_t, c_void_p]),
    "utv_randutv_step_bufsize": (c_size_t, [c_int, c_int, c_int, c_int, c_int]),
    "utv_randutv_step_f64": (c_int, [c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_void_p,
                                     c_long, c_void_p, c_long, c_void_p, c_long, c_void_p, c_long,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_size_t, c_void_p]),
    "utv_randutv_basic_f32_bufsize": (c_size_t, [c_int, c_int, c_int, c_int]),
    "utv_randutv_basic_f32": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_long, c_void_p,
                                      c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "utv_powerurv_bufsize": (c_size_t, [c_int, c_int, c_int]),
    "utv_powerurv_f64": (c_int, [c_int, c_int, c_int, c_void_p, c_long, c_void_p, c_long,
                                 c_void_p, c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                 c_long, c_void_p, c_long, c_void_p, c_size_t, c_void_p]),
    "utv_powerurv_f64_ev": (c_int, [c_int, c_int, c_int, c_void_p, c_long, c_void_p, c_long,
                                 c_void_p, c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                 c_long, c_void_p, c_long, c_void_p, c_size_t, c_void_p, c_void_p,
                                 c_void_p]),
    "utv_powerurv_f64_yhat": (c_int, [c_int, c_int, c_int, c_void_p, c_long, c_void_p, c_long,
                                   c_void_p, c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                   c_long, c_void_p, c_long, c_void_p, c_size_t, c_void_p,
                                   c_void_p, c_void_p]),
    "utv_powerurv_f64_cols": (c_int, [c_int, c_int, c_int, c_void_p, c_long, c_void_p, c_long,
                                      c_void_p, c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                      c_long, c_void_p, c_long, c_void_p, c_long, c_void_p, c_size_t,
                                      c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                      c_void_p]),
    "utv_dgeqrf_rows_max": (c_int, []),
    "utv_dgeqp3_bufsize": (c_size_t, [c_int, c_int]),
    "utv_dgeqp3_max_dim": (c_int, []),
    "utv_dgeqp3_f64": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_long, c_void_p, c_long,
                               c_void_p, c_long, c_void_p, c_void_p, c_size_t, c_void_p]),
    "utv_sgemm_tf32x3": (c_int, [c_char, c_char, c_int, c_int, c_int, ctypes.c_float, c_void_p, c_long,
                                 c_void_p, c_long, ctypes.c_float, c_void_p, c_long, c_void_p]),
    "utv_dlacpy": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_long, c_void_p]),
    "utv_dlaset": (c_int, [c_char, c_int, c_int, c_double, c_double, c_void_p, c_long, c_void_p]),
    "utv_slaset": (c_int, [c_char, c_int, c_int, ctypes.c_float, ctypes.c_float, c_void_p, c_long,
                           c_void_p]),
    "utv_dnonfinite": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_void_p]),
    "utv_zero": (c_int, [c_void_p, c_size_t, c_void_p]),
    "utv_dtri_zero": (c_int, [c_char, c_int, c_int, c_void_p, c_long, c_void_p]),
    "utv_dtranspose": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_long, c_void_p]),
    "utv_dgen_bie": (c_int, [c_int, c_void_p, c_long, c_void_p]),
    "utv_dgen_kahan": (c_int, [c_int, c_double, c_void_p, c_long, c_void_p]),
    "utv_dtrailing_fro_bufsize": (c_size_t, [c_int, c_int]),
    "utv_dtrailing_fro": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_void_p, c_size_t,
                                  c_void_p]),
    "utv_ddiag_scale": (c_int, [c_char, c_int, c_int, c_void_p, c_double, c_void_p, c_long,
                                c_void_p]),
    "utv_dgetrf_signed_bufsize": (c_size_t, [c_int, c_int]),
    "utv_dgetrf_signed": (c_int, [c_int, c_int, c_void_p, c_long, c_void_p, c_void_p, c_size_t,
                                  c_void_p]),
    "utv_dtrsm_bufsize": (c_size_t, [c_int, c_int]),
    "utv_dtrsm_right": (c_int, [c_char, c_char, c_char, c_int, c_int, c_void_p, c_long, c_void_p,
                                c_long, c_void_p, c_size_t, c_void_p]),
    "utv_comm_nccl_available": (c_int, []),
    "utv_comm_nccl_unique_id": (c_int, [c_void_p]),
    "utv_comm_init_nccl": (c_int, [c_void_p, c_int, c_int, c_void_p]),
    "utv_comm_from_nccl": (c_int, [c_void_p, c_void_p]),
    "utv_comm_init_local": (c_int, [c_int, c_void_p]),
    "utv_comm_rank": (c_int, [c_void_p]),
    "utv_comm_size": (c_int, [c_void_p]),
    "utv_comm_destroy": (c_int, [c_void_p]),
    "utv_comm_allreduce_sum_f64": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "utv_comm_allgather_f64": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "utv_comm_broadcast_f64": (c_int, [c_void_p, c_void_p, c_size_t, c_int, c_void_p]),
    "utv_powerurv_sharded_bufsize": (c_size_t, [c_int, c_int, c_int, c_int]),
    "utv_powerurv_sharded_f64": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_long, c_void_p,
                                         c_long, c_void_p, c_long, c_void_p, c_long, c_void_p,
                                         c_long, c_void_p, c_long, c_void_p, c_long, c_int,
                                         c_void_p, c_size_t, c_void_p]),
    "utv_launch_count": (ctypes.c_longlong, []),
    "utv_profile_begin": (None, []),
    "utv_profile_end": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "utv_profile_busy": (c_int, [c_void_p]),
    "utv_rng_set_tables": (c_int, [c_void_p, c_void_p, c_void_p]),
    "utv_rng_pcg64_normals": (c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                      c_void_p, ctypes.c_uint64, c_int, c_void_p]),
}

PROF_CATEGORIES = ("dgemm_dmma", "splitk_reduce", "panel_qr", "jacobi_rounds",
                   "jacobi_finish", "small_ops", "sgemm_tf32x3", "qrcp")


def load():
    """Load libutvb200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libutvb200.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2106_13402_b200.build` (no CPU fallback exists)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class UtvError(RuntimeError):
    pass


def check(status, what):
    if status != 0:
        raise UtvError(f"{what} failed with status {status}")


# ---------------------------------------------------------------------------
# device matrices
# ---------------------------------------------------------------------------

def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2106_13402_b200 needs a CUDA device (B200); no CPU fallback")
    return torch


def even_ld(rows):
    return max(2, rows + (rows & 1))


@dataclass
class DMat:
    """Column-major FP64 device matrix: a view into a torch tensor of shape
    (cols_total, ld) starting at element offset `off`."""
    t: object
    rows: int
    cols: int
    ld: int
    off: int = 0

    @property
    def esize(self):
        return self.t.element_size()

    @property
    def ptr(self):
        return self.t.data_ptr() + self.esize * self.off

    def at(self, r, c):
        return self.ptr + self.esize * (r + c * self.ld)

    def sub(self, r0, c0, nr, nc):
        """View of rows r0:r0+nr, columns c0:c0+nc (no copy)."""
        if r0 < 0 or c0 < 0 or r0 + nr > self.rows or c0 + nc > self.cols:
            raise IndexError("DMat.sub out of range")
        return DMat(self.t, nr, nc, self.ld, self.off + r0 + c0 * self.ld)

    def tensor(self):
        """(cols, rows) strided torch view of the block (column j = row j of the view)."""
        return self.t.as_strided((self.cols, self.rows), (self.ld, 1),
                                 self.t.storage_offset() + self.off)

    def to_numpy(self):
        """Host copy as an F-order numpy array (staged through pinned memory
        for large contiguous blocks, see d2h_numpy)."""
        if self.off == 0 and self.ld == self.rows and self.rows * self.cols * self.esize >= (8 << 20):
            return d2h_numpy(self)
        host = self.tensor().cpu().numpy()              # (cols, rows) C order
        return host.T                                   # (rows, cols) F order


# ---------------------------------------------------------------------------
# host <-> device staging
# ---------------------------------------------------------------------------
# Pageable device->host copies run at ~2 GB/s on the B200 hosts; a DMA into a
# small pinned ring (~50 GB/s) overlapped with multi-threaded host memcpy
# into the destination numpy array is several times faster and needs no
# large page-locked allocation.
_RING = None
# The pinned staging rings are process-wide; the public API is re-entrant
# (utvkit's functions are pure), so each ring is used under its own lock —
# concurrent calls from several host threads serialise their staging.
_RING_LOCK = threading.Lock()
# One device pipeline at a time: the drivers share library-owned side
# streams, events and tile-scheduler slots, so public calls made from
# several host threads run one after another (re-entrant: rurv -> power_urv).
_API_LOCK = threading.RLock()


def serialized(fn):
    import functools

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        with _API_LOCK:
            return fn(*args, **kwargs)
    return wrapper

_H2D_LOCK = threading.Lock()
_ASYNC_LOCK = threading.Lock()
_RING_CHUNK = 64 << 20
_POOL = None


def _ring():
    global _RING, _POOL
    if _RING is None:
        import concurrent.futures

        import torch
        _RING = [(torch.empty(_RING_CHUNK, dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
                 for _ in range(3)]
        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=8)
    return _RING, _POOL


def _d2h_bytes(src, dst, stream, ring, pool, nthr=8):
    """Device bytes `src` (torch uint8) -> host bytes `dst` (numpy uint8),
    staged through the pinned `ring` (DMA on `stream`) with an nthr-way
    host memcpy per chunk, chunks pipelined against each other."""
    nb = dst.nbytes
    chunks = [(off, min(_RING_CHUNK, nb - off)) for off in range(0, nb, _RING_CHUNK)]

    def copy_out(k, off, sz):
        buf = ring[k][0].numpy()
        step = (sz + nthr - 1) // nthr

        def part(lo, hi):
            dst[off + lo: off + hi] = buf[lo:hi]
        futs = [pool.submit(part, j * step, min(sz, (j + 1) * step)) for j in range(nthr) if j * step < sz]
        for f in futs:
            f.result()

    pending = []
    for i, (off, sz) in enumerate(chunks):
        k = i % len(ring)
        if len(pending) == len(ring):          # ring full: drain the oldest chunk
            j, o, z = pending.pop(0)
            ring[j][1].synchronize()
            copy_out(j, o, z)
        ring[k][0][:sz].copy_(src[off:off + sz], non_blocking=True)
        ring[k][1].record(stream)
        pending.append((k, off, sz))
    for j, o, z in pending:
        ring[j][1].synchronize()
        copy_out(j, o, z)


_H2D_RING = None


def _h2d_bytes(src, dst, stream, nthr=8):
    """Host bytes `src` (numpy uint8) -> device bytes `dst` (torch uint8):
    an nthr-way host memcpy into a pinned ring buffer, then its DMA on
    `stream`, chunks pipelined so the memcpy of chunk i+1 overlaps the DMA
    of chunk i (a pageable copy_ runs at ~10 GB/s on the B200 hosts)."""
    with _H2D_LOCK:
        _h2d_bytes_locked(src, dst, stream, nthr)


def _h2d_bytes_locked(src, dst, stream, nthr):
    global _H2D_RING
    import torch
    if _H2D_RING is None:
        _H2D_RING = [(torch.empty(_RING_CHUNK, dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
                     for _ in range(3)]
    ring = _H2D_RING
    _, pool = _ring()
    nb = src.nbytes
    for i, off in enumerate(range(0, nb, _RING_CHUNK)):
        sz = min(_RING_CHUNK, nb - off)
        buf, ev = ring[i % len(ring)]
        ev.synchronize()                       # this buffer's previous DMA is done
        host = buf.numpy()
        step = (sz + nthr - 1) // nthr

        def part(lo, hi, host=host, off=off):
            host[lo:hi] = src[off + lo: off + hi]
        futs = [pool.submit(part, j * step, min(sz, (j + 1) * step)) for j in range(nthr) if j * step < sz]
        for f in futs:
            f.result()
        with torch.cuda.stream(stream):
            dst[off:off + sz].copy_(buf[:sz], non_blocking=True)
            ev.record(stream)


def h2d_numpy(a, m):
    """F-order numpy array -> contiguous (ld == rows) device block `m`."""
    import torch
    flat = a.reshape(-1, order="F").view(np.uint8)
    dst = m.t.view(-1)[m.off: m.off + m.rows * m.cols].view(torch.uint8)
    _h2d_bytes(flat, dst, torch.cuda.current_stream())


def d2h_numpy(m):
    """Contiguous (ld == rows) device block -> new F-order numpy array."""
    import torch
    ring, pool = _ring()
    dt = np.float64 if m.t.dtype == torch.float64 else np.float32
    out = np.empty((m.rows, m.cols), dtype=dt, order="F")
    dst = out.reshape(-1, order="F").view(np.uint8)
    src = m.t.view(-1)[m.off: m.off + m.rows * m.cols].view(torch.uint8)
    with _RING_LOCK:
        _d2h_bytes(src, dst, torch.cuda.current_stream(), ring, pool)
    return out


_D2H_TRACE = bool(os.environ.get("UTV_D2H_TRACE"))
_D2H_T0 = __import__("time").perf_counter()


class AsyncD2H:
    """Background device->host copies of column blocks that are FINAL (no
    later kernel writes them): each job waits (on the device) for an event
    of the compute stream, then streams the blocks through a private pinned
    ring on a private copy stream into preallocated F-order numpy arrays, so
    results leave the GPU while the factorisation is still running."""

    _shared = {}

    def __init__(self):
        import queue
        import threading

        import torch
        if "ring" not in AsyncD2H._shared:
            AsyncD2H._shared["ring"] = [(torch.empty(_RING_CHUNK, dtype=torch.uint8, pin_memory=True),
                                         torch.cuda.Event()) for _ in range(3)]
        self.ring = AsyncD2H._shared["ring"]
        _, self.pool = _ring()
        self.stream = torch.cuda.Stream()
        self.q = queue.Queue()
        self.err = None
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()

    def push(self, event, blocks):
        """blocks: list of (DMat with ld == rows, host F-order array, c0, c1)."""
        self.q.put((event, blocks))

    _fault_pool = None

    def prefault(self, arrays, chunk=_RING_CHUNK):
        """Touch every page of the (fresh, np.empty) destination arrays on
        background threads while the device computes: a first-touch write
        into new anonymous memory runs at a fraction of the bandwidth of a
        write into mapped pages, so the later copies out of the pinned ring
        (the tail of the timed call) no longer pay the page faults.  Chunks
        are queued round-robin over the arrays in column order, the order
        the results become final."""
        import concurrent.futures
        if AsyncD2H._fault_pool is None:
            AsyncD2H._fault_pool = concurrent.futures.ThreadPoolExecutor(max_workers=4)
        flat = [a.reshape(-1, order="F").view(np.uint8) for a in arrays]
        self.faults = getattr(self, "faults", {})
        for a in arrays:
            self.faults.setdefault(id(a), [])
        nchunks = max(-(-f.nbytes // chunk) for f in flat)
        for k in range(nchunks):
            for a, f in zip(arrays, flat):
                lo = k * chunk
                if lo >= f.nbytes:
                    continue
                hi = min(f.nbytes, lo + chunk)
                fut = AsyncD2H._fault_pool.submit(f[lo:hi].fill, 0)
                self.faults[id(a)].append((lo, hi, fut))

    def _wait_faults(self, host, lo, hi):
        for flo, fhi, fut in getattr(self, "faults", {}).get(id(host), ()):
            if flo < hi and fhi > lo:
                fut.result()

    def _run(self):
        import torch
        while True:
            job = self.q.get()
            if job is None:
                return
            if self.err is not None:
                continue
            event, blocks = job
            try:
                # wait for the producing kernels on the host BEFORE taking the
                # shared ring: a job whose data is not final yet must not
                # hold the ring (and every other copy) while it waits
                event.synchronize()
                if _D2H_TRACE:
                    import time
                    t1 = time.perf_counter()
                with torch.cuda.stream(self.stream):
                    self.stream.wait_event(event)
                    for m, host, c0, c1 in blocks:
                        if c1 <= c0:
                            continue
                        es = m.esize
                        src = m.t.view(-1)[m.off + c0 * m.ld: m.off + c1 * m.ld].view(torch.uint8)
                        dst = host.reshape(-1, order="F")[c0 * m.rows: c1 * m.rows].view(np.uint8)
                        assert m.ld == m.rows and dst.nbytes == src.numel() and es == host.itemsize
                        self._wait_faults(host, c0 * m.rows * es, c1 * m.rows * es)
                        with _ASYNC_LOCK:
                            _d2h_bytes(src, dst, self.stream, self.ring, self.pool)
                if _D2H_TRACE:
                    t2 = time.perf_counter()
                    nb = sum((c1 - c0) * m.rows * m.esize for m, _, c0, c1 in blocks)
                    print(f"[d2h {id(self) % 1000:3d}] ready {t1 - _D2H_T0:.3f} copied {t2 - _D2H_T0:.3f} "
                          f"{nb / 2**20:.0f} MiB {nb / max(t2 - t1, 1e-9) / 1e9:.1f} GB/s", flush=True)
            except BaseException as e:  # surfaced by finish()
                self.err = e

    def finish(self):
        self.q.put(None)
        self.th.join()
        if self.err is not None:
            raise self.err


def dempty(rows, cols, ld=None, dtype=None):
    torch = torch_cuda()
    dtype = torch.float64 if dtype is None else dtype
    if ld is None:
        # fp64: even ld (TMA 16-byte strides); fp32: multiple of 4
        ld = even_ld(rows) if dtype == torch.float64 else max(4, (rows + 3) // 4 * 4)
    t = torch.empty((max(cols, 1), ld), dtype=dtype, device="cuda")
    return DMat(t, rows, cols, ld)


def _laset(m, alpha, beta):
    check(load().utv_dlaset(b"A", m.rows, m.cols, alpha, beta, m.ptr, m.ld, stream_ptr()),
          "utv_dlaset")
    return m


def dzero_vec(n, dtype=None):
    """n zeros on the device (cudaMemsetAsync through utv_zero, no torch kernel)."""
    torch = torch_cuda()
    v = torch.empty(max(int(n), 1), dtype=torch.float64 if dtype is None else dtype, device="cuda")
    check(load().utv_zero(v.data_ptr(), v.numel() * v.element_size(), stream_ptr()), "utv_zero")
    return v[: int(n)] if n else v[:0]


def dzeros(rows, cols):
    return _laset(dempty(rows, cols), 0.0, 0.0)


def deye(n):
    return _laset(dempty(n, n), 0.0, 1.0)


def dfrom_numpy(a, pinned=False, dtype=None):
    """Copy a 2-D array to the device (column-major; float64 unless dtype=float32)."""
    torch = torch_cuda()
    npdt = np.float32 if dtype == torch.float32 else np.float64
    a = np.asfortranarray(a, dtype=npdt)
    rows, cols = a.shape
    m = dempty(rows, cols, dtype=torch.float32 if npdt == np.float32 else torch.float64)
    if not pinned and m.ld == rows and a.nbytes >= (8 << 20):
        h2d_numpy(a, m)
        return m
    src = torch.from_numpy(a.T)             # (cols, rows) view of the F-order data
    if pinned:
        src = src.pin_memory()
    m.t[:cols, :rows].copy_(src, non_blocking=pinned)
    return m


def workspace(nbytes):
    torch = torch_cuda()
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")


def stream_ptr():
    torch = torch_cuda()
    return torch.cuda.current_stream().cuda_stream


def profile_begin():
    load().utv_profile_begin()


def profile_end():
    """Synchronise and return {category: dict(ms, flops, bytes, count)}."""
    n = len(PROF_CATEGORIES)
    ms = (ctypes.c_double * n)()
    fl = (ctypes.c_double * n)()
    by = (ctypes.c_double * n)()
    ct = (ctypes.c_longlong * n)()
    load().utv_profile_end(ms, fl, by, ct)
    busy = (ctypes.c_double * n)()
    load().utv_profile_busy(busy)
    return {PROF_CATEGORIES[i]: dict(ms=ms[i], busy_ms=busy[i], flops=fl[i], bytes=by[i],
                                     count=int(ct[i]))
            for i in range(n)}


def launch_count():
    return int(load().utv_launch_count())
