"""C1-style single-array stream shuffles under each eligible kernel (dev tool)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_06213_b200 as B

for n in (1000, 10000, 50000):
    z = torch.arange(n, dtype=torch.int32, device="cuda")
    for kern in ("", "hash"):
        os.environ["BR_SHUFFLE_KERNEL"] = kern
        s = B.Pcg64Source(42)
        for _ in range(3):
            B.shuffle_batched(s, z)
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); B.shuffle_batched(s, z); b.record(); b.synchronize()
            ts.append(a.elapsed_time(b))
        print(n, kern or "default", B.last_kernel(), round(statistics.median(ts), 4), "ms (call incl. state round trip)")
