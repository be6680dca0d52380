"""Bulk roll throughput for k = 1..8 (dev tool): ms per call and HBM fraction."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_06213_b200 as B

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6542.7
KS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else (1, 2, 3, 4, 5, 6, 8)
for k in KS:
    nb = (1 << 26) // k
    span = {1: 1 << 30, 2: 1 << 16, 3: 1 << 10, 4: 1 << 10, 5: 4000, 6: 1000, 8: 200}[k]
    bounds = (torch.randint(0, span - 2, (nb * k,), dtype=torch.int64, device="cuda") + 2).to(torch.int32)
    ds = B.DeviceStream(5)
    rolls = torch.empty(nb * k, dtype=torch.int32, device="cuda")
    words = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        B.roll_batches(ds, bounds, k, out=(rolls, words), check=False)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); B.roll_batches(ds, bounds, k, out=(rolls, words), check=False); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    byt = nb * (8 * k + 1)
    print(f"k={k} nb={nb} {ms:.3f} ms  {nb * k / ms / 1e6:.1f} G rolls/s  {byt / ms / 1e6:.0f} GB/s = {byt / ms / 1e6 / peak:.2f} of HBM  {B.last_kernel()}")
