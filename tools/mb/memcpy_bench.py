"""Host memcpy bandwidth into pinned memory (single thread and threads)."""
import time
import threading
import numpy as np
import torch

n = 3_407_872
src = np.random.randint(0, 1 << 40, n // 8, dtype=np.int64).view(np.uint8)
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()
dst2 = np.empty(n, dtype=np.uint8)
for name, d in (("pinned", dst), ("pageable", dst2)):
    for _ in range(3):
        np.copyto(d, src)
    t = time.perf_counter()
    for _ in range(20):
        np.copyto(d, src)
    dt = (time.perf_counter() - t) / 20
    print(f"{name} 1 thread: {n / dt / 1e9:.1f} GB/s ({dt * 1e6:.0f} us)")


def par(d, k):
    pieces = np.array_split(np.arange(n), k)
    def work(p):
        np.copyto(d[p[0]:p[-1] + 1], src[p[0]:p[-1] + 1])
    ts = [threading.Thread(target=work, args=(p,)) for p in pieces]
    t = time.perf_counter()
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    return time.perf_counter() - t


for k in (2, 4, 8):
    dt = min(par(dst, k) for _ in range(10))
    print(f"pinned {k} threads: {n / dt / 1e9:.1f} GB/s ({dt * 1e6:.0f} us)")
import os
print("cpus", os.cpu_count())
