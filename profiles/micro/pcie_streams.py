"""PCIe probe (experiment): pinned H2D throughput with 1/2/4/8 concurrent
copies of one 8 GiB transfer (split into equal parts on separate streams), with
and without a concurrent 4 GiB D2H."""
import time

import torch

n = 8 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
m = 4 << 30
ho = torch.empty(m, dtype=torch.uint8).pin_memory()
do = torch.empty(m, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(9)]


def run(k, with_d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    part = n // k
    for i in range(k):
        with torch.cuda.stream(streams[i]):
            d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
    if with_d2h:
        with torch.cuda.stream(streams[8]):
            ho.copy_(do, non_blocking=True)
    ev = []
    for i in range(k):
        e = torch.cuda.Event()
        e.record(streams[i])
        ev.append(e)
    for e in ev:
        e.synchronize()
    t_h2d = time.perf_counter() - t0
    torch.cuda.synchronize()
    return n / t_h2d / 1e9, (time.perf_counter() - t0)


for with_d2h in (False, True):
    for k in (1, 2, 4, 8):
        run(k, with_d2h)
        bw, tt = run(k, with_d2h)
        print(f"H2D x{k} {'+ D2H' if with_d2h else '     '}: H2D {bw:.1f} GB/s (all done {tt*1e3:.0f} ms)", flush=True)
