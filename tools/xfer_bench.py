"""Host<->device transfer options for 2 GiB numpy arrays."""
import sys, time, threading
sys.path.insert(0, '.')
import numpy as np
import torch
t = time.perf_counter
n = 16384
a = np.asfortranarray(np.random.default_rng(0).standard_normal((n, n)))
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for rep in range(2):
    T0 = t(); d.copy_(torch.from_numpy(a.T)); torch.cuda.synchronize(); print("pageable copy_", t() - T0, flush=True)
T0 = t(); p = torch.empty((n, n), dtype=torch.float64, pin_memory=True); print("pinned alloc 2GiB", t() - T0, flush=True)
T0 = t(); p.numpy()[...] = a.T; print("memcpy to pinned (1 thread)", t() - T0, flush=True)
T0 = t(); d.copy_(p, non_blocking=True); torch.cuda.synchronize(); print("pinned H2D", t() - T0, flush=True)
T0 = t(); p.copy_(d, non_blocking=True); torch.cuda.synchronize(); print("pinned D2H", t() - T0, flush=True)
T0 = t(); h = d.cpu(); print("pageable D2H .cpu()", t() - T0, flush=True)
# cudaHostRegister on the numpy buffer
cudart = torch.cuda.cudart()
T0 = t(); r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0); print("hostRegister", t() - T0, r, flush=True)
T0 = t(); d.copy_(torch.from_numpy(a.T), non_blocking=True); torch.cuda.synchronize(); print("registered H2D", t() - T0, flush=True)
T0 = t(); cudart.cudaHostUnregister(a.ctypes.data); print("unregister", t() - T0, flush=True)
# multi-threaded chunked staging through a small pinned ring
def staged_h2d(src, dst, chunk=64 << 20, nthr=8):
    flat_src = src.reshape(-1).view(np.uint8) if src.flags['C_CONTIGUOUS'] else src.T.reshape(-1).view(np.uint8)
    nb = flat_src.nbytes
    bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
    evs = [torch.cuda.Event() for _ in range(4)]
    dflat = dst.view(-1).view(torch.uint8)
    st = torch.cuda.Stream()
    i = 0
    for off in range(0, nb, chunk):
        k = i % 4
        evs[k].synchronize()
        sz = min(chunk, nb - off)
        bnp = bufs[k].numpy()
        def cp(lo, hi):
            bnp[lo:hi] = flat_src[off + lo: off + hi]
        step = (sz + nthr - 1) // nthr
        ths = [threading.Thread(target=cp, args=(j * step, min(sz, (j + 1) * step))) for j in range(nthr)]
        [x.start() for x in ths]; [x.join() for x in ths]
        with torch.cuda.stream(st):
            dflat[off:off + sz].copy_(bufs[k][:sz], non_blocking=True)
            evs[k].record(st)
        i += 1
    st.synchronize()
T0 = t(); staged_h2d(a, d); print("staged 8-thread H2D", t() - T0, flush=True)
print("check", torch.equal(d.cpu(), torch.from_numpy(a.T)))
