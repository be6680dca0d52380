"""Cost of the roll fixup per resolved rejection (dev tool): batches of k = 2 with tiny
products except R evenly spaced heavy batches (product 2^63 + 1: each rejects its first word
with probability ~1/2), timed for several R and run lengths."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2408_06213_b200 as B

k = 2
for nb in (1 << 20, 1 << 24):
    for R in (0, 100, 1000, 4000):
        b = torch.full((nb, k), 3, dtype=torch.int64)
        if R:
            idx = torch.linspace(10, nb - 10, R).long()
            b[idx, 0] = 0xFFFFFFFF
            b[idx, 1] = 0x80000001  # product ~2^63: rejects ~1/2
        bounds = b.reshape(-1).to(torch.int32).cuda()
        ds = B.DeviceStream(11)
        rolls = torch.empty(nb * k, dtype=torch.int32, device="cuda")
        words = torch.empty(nb, dtype=torch.uint8, device="cuda")
        for _ in range(2):
            B.roll_batches(ds, bounds, k, out=(rolls, words), check=False)
        ts, rej = [], []
        for _ in range(5):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); B.roll_batches(ds, bounds, k, out=(rolls, words), check=False); e.record(); e.synchronize()
            ts.append(a.elapsed_time(e))
            rej.append(int((words > 1).sum()))
        ms = statistics.median(ts)
        nrej = statistics.median(rej)
        line = f"nb={nb:>9} R={R:>5} rejected batches ~{nrej:>5}  {ms:8.3f} ms  {(ms * 1e3 / nrej) if nrej else 0:6.2f} us/rejection"
        if os.environ.get("BR_LIB") and R:  # BR_FIXUP_PROF build (tools/fixup_prof.sh): block 0's phase times
            pr = ds.workspace[88:120].cpu().view(torch.int64).tolist()
            it = max(pr[3], 1)
            line += f"  | per iteration: re-run {pr[0] / it / 1e3:.2f} us, barrier {pr[1] / it / 1e3:.2f} us, records {pr[2] / it / 1e3:.2f} us ({pr[3]} it)"
        print(line)
