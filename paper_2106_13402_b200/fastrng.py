"""Parallel, bit-identical reproduction of the reference's Gaussian stream.

The reference draws G with numpy ``Generator(PCG64(seed)).standard_normal``
(utvkit matrix.py:16-33) — a sequential stream (~10 ns per normal on these
hosts, 2.8 s for powerURV's 16384^2 G).  ``libutvb200``'s
``utv_rng_pcg64_normals`` (csrc/rng_host.cu) generates the same numbers on
all host cores: PCG64 jump-ahead to chunk starts, speculative ziggurat parses
stitched at the first common normal boundary, numpy's own ziggurat tables and
libm calls.  Before first use the native path is checked against numpy on
several seeds (values AND the generator state afterwards); any disagreement,
a missing table or a failed stitch falls back to numpy itself, so the stream
the caller sees is always exactly the reference's.
"""

import ctypes
import os
import struct
import threading

import numpy as np

_MIN_PARALLEL = 1 << 18      # below this, numpy's own loop is as fast
_lock = threading.Lock()
_state = {"ok": None}


def _ziggurat_tables():
    """numpy's (ki, wi, fi) double-precision normal ziggurat tables, read from
    the installed numpy binary (layout fi | wi | ki, located by ki[0..2])."""
    import numpy.random._generator as gmod
    blob = open(gmod.__file__, "rb").read()
    sig = struct.pack("<QQQ", 0x000EF33D8025EF6A, 0, 0x000C08BE98FBC6A8)
    at = blob.find(sig)
    if at < 4096:
        return None
    ki = np.frombuffer(blob, dtype=np.uint64, count=256, offset=at).copy()
    wi = np.frombuffer(blob, dtype=np.float64, count=256, offset=at - 2048).copy()
    fi = np.frombuffer(blob, dtype=np.float64, count=256, offset=at - 4096).copy()
    if not (fi[0] == 1.0 and np.all(np.diff(fi) < 0) and np.all(np.diff(wi[1:]) > 0)):
        return None
    return ki, wi, fi


def _native(gen, out):
    """Fill `out` (C-contiguous float64) from `gen` natively; advance gen. True on success."""
    from ._lib import load
    lib = load()
    st = gen.bit_generator.state
    if st.get("bit_generator") != "PCG64" or st.get("has_uint32", 0):
        return False
    s, inc = st["state"]["state"], st["state"]["inc"]
    m64 = (1 << 64) - 1
    used = ctypes.c_uint64(0)
    rc = lib.utv_rng_pcg64_normals(s >> 64, s & m64, inc >> 64, inc & m64,
                                   out.ctypes.data_as(ctypes.c_void_p), out.size,
                                   os.cpu_count() or 1, ctypes.byref(used))
    if rc != 0:
        return False
    gen.bit_generator.advance(int(used.value))
    return True


def _enable():
    from ._lib import load
    lib = load()
    tabs = _ziggurat_tables()
    if tabs is None:
        return False
    ki, wi, fi = tabs
    lib.utv_rng_set_tables(ki.ctypes.data_as(ctypes.c_void_p), wi.ctypes.data_as(ctypes.c_void_p),
                           fi.ctypes.data_as(ctypes.c_void_p))
    for seed, count in ((0, 300_007), (12345, 1 << 20), (2 ** 63 + 7, 70_001)):
        ref = np.random.Generator(np.random.PCG64(seed))
        mine = np.random.Generator(np.random.PCG64(seed))
        want = ref.standard_normal(count)
        got = np.empty(count)
        if not _native(mine, got) or not np.array_equal(got.view(np.uint64), want.view(np.uint64)):
            return False
        if mine.bit_generator.state != ref.bit_generator.state:
            return False
    return True


def enabled():
    with _lock:
        if _state["ok"] is None:
            try:
                _state["ok"] = bool(_enable())
            except Exception:
                _state["ok"] = False
        return _state["ok"]


def standard_normal_into(gen, out):
    """gen.standard_normal(out.shape, out=out) — same values, same final state."""
    if out.size >= _MIN_PARALLEL and out.flags.c_contiguous and out.dtype == np.float64 \
            and enabled() and _native(gen, out.reshape(-1)):
        return out
    gen.standard_normal(out.shape, out=out)
    return out


def standard_normal(gen, shape):
    out = np.empty(shape)
    return standard_normal_into(gen, out)
