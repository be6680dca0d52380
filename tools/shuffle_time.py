"""Times shuffle_many on a BASELINE shape for each kernel named on the command line
(BR_SHUFFLE_KERNEL values; 'default' = the dispatcher's pick).  Dev tool (A/B timing).
  python tools/shuffle_time.py c5 default large stage"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import __graft_entry__

__graft_entry__.build()
import paper_2408_06213_b200 as B

CFG = {"c3": (64, 1 << 20, 4, 1234), "c4": (4096, 1 << 16, 4, 99), "c5": (1 << 20, 256, 8, 5)}
n, na, eb, seed = CFG[sys.argv[1]]
reps = int(os.environ.get("REPS", "5"))
for kern in sys.argv[2:]:
    if kern == "default":
        os.environ.pop("BR_SHUFFLE_KERNEL", None)
    else:
        os.environ["BR_SHUFFLE_KERNEL"] = kern
    data = B.pcg64_fill(seed, n * na) if eb == 8 else torch.arange(n, dtype=torch.int32, device="cuda").repeat(na)
    B.shuffle_many(data, n, seed)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        B.shuffle_many(data, n, seed)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"{sys.argv[1]} {kern:8s} {B.last_kernel():40s} median {statistics.median(ts):.3f} ms  min {min(ts):.3f}",
          flush=True)
