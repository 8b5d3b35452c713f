"""Host memory bandwidth of the box: T threads each widening a uint16 array
into uint32 (read 2 B, write 4 B per element -- the shape of a host-side id
decode) and plain copies, aggregate GB/s."""
import os
import sys
import threading
import time

import numpy as np

T = int(sys.argv[1]) if len(sys.argv) > 1 else os.cpu_count()
N = 1 << 27   # elements per thread


def run(fn, nbytes):
    ths = [threading.Thread(target=fn, args=(i,)) for i in range(T)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    return nbytes * T / dt / 1e9


src16 = [np.ones(N, np.uint16) for _ in range(T)]
dst32 = [np.zeros(N, np.uint32) for _ in range(T)]
src32 = [np.ones(N, np.uint32) for _ in range(T)]


def widen(i):
    np.bitwise_or(src16[i], np.uint32(0x10000), out=dst32[i], casting="unsafe")


def copy(i):
    np.copyto(dst32[i], src32[i])


for name, fn, nb in (("widen u16->u32 (6 B/elem)", widen, 6 * N), ("copy u32 (8 B/elem)", copy, 8 * N)):
    best = max(run(fn, nb) for _ in range(3))
    print(f"{name}: {best:.1f} GB/s aggregate on {T} threads ({best / (nb / N) :.2f} G elem/s)")
