"""C5 shape with a varying number of arrays: how the stage kernel's one-CTA-per-array grid
fills 148 SMs x 2 CTAs (dev tool; prints ms per call and elements/s)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2408_06213_b200 as B

n = 1 << 20
for na in [int(x) for x in sys.argv[1:]] or [74, 148, 222, 256, 296]:
    data = B.pcg64_fill(5, n * na)
    B.shuffle_many(data, n, 5)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        B.shuffle_many(data, n, 5)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = statistics.median(ts)
    print(f"arrays {na:4d}  {B.last_kernel():28s} {t:7.3f} ms  {na * n / t / 1e6:7.2f} G elements/s", flush=True)
    del data
