"""Host->device upload paths for large pageable numpy arrays (dev tool):
pageable cudaMemcpy, cudaHostRegister + copy (+ unregister), and chunked
multi-threaded staging through pinned buffers.

  python tools/h2d_probe.py [GB]
"""
import ctypes
import os
import sys
import threading
import time

import numpy as np
import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 1.6
n = int(gb * 2**30 / 8)
src = np.random.default_rng(0).random(n)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
cudart = torch.cuda.cudart()
print("cpus", os.cpu_count(), "GB", gb)


def timeit(name, fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"{name:28s} {best * 1e3:8.1f} ms  {gb / best:6.1f} GB/s", flush=True)


def pageable():
    dev.copy_(torch.from_numpy(src), non_blocking=False)


def registered():
    ptr, size = src.ctypes.data, src.nbytes
    assert cudart.cudaHostRegister(ptr, size, 0) == 0
    dev.copy_(torch.from_numpy(src), non_blocking=True)
    torch.cuda.synchronize()
    cudart.cudaHostUnregister(ptr)


CH = 64 << 20
pins = [torch.empty(CH // 8, dtype=torch.float64).pin_memory() for _ in range(16)]


def staged(threads):
    def run():
        s = torch.cuda.Stream()
        nch = (src.nbytes + CH - 1) // CH
        evs = [None] * len(pins)
        lock = threading.Lock()
        nxt = [0]

        def worker(w):
            while True:
                with lock:
                    c = nxt[0]
                    nxt[0] += 1
                if c >= nch:
                    return
                b = c % len(pins)
                e = evs[b]
                if e is not None:
                    e.synchronize()
                lo = c * (CH // 8)
                hi = min(n, lo + CH // 8)
                pins[b][: hi - lo].numpy()[:] = src[lo:hi]
                with torch.cuda.stream(s):
                    dev[lo:hi].copy_(pins[b][: hi - lo], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(s)
                evs[b] = ev

        ts = [threading.Thread(target=worker, args=(w,)) for w in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        s.synchronize()
    return run


timeit("pageable copy", pageable)
timeit("cudaHostRegister + copy", registered)
for t in (1, 4, 8):
    timeit(f"pinned staging x{t} threads", staged(t))
assert torch.equal(dev.cpu(), torch.from_numpy(src))
