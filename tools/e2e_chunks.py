"""e2e C2 through roll_batches with host pinned buffers, for several chunk counts (dev tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2408_06213_b200 as B

nb = bench.NB_C2
bounds, stream, rolls, words = bench.setup_c2(torch, B, 0, nb)
hb = bounds.cpu().pin_memory()
hr = torch.empty(2 * nb, dtype=torch.int32).pin_memory()
hw = torch.empty(nb, dtype=torch.uint8).pin_memory()
for ch in [int(x) for x in sys.argv[1:]] or (4, 8, 16, 32, 64):
    B.roll_batches(stream, hb, 2, out=(hr, hw), chunks=ch)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        B.roll_batches(stream, hb, 2, out=(hr, hw), chunks=ch, check=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"chunks {ch}: {ms:.3f} ms/step, {2 * nb / ms / 1e6:.2f} G rolls/s")
