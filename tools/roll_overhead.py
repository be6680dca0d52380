"""Measure the per-step overhead of the roll fixup launch (dev tool)."""
import ctypes as C
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2408_06213_b200 as B
from paper_2408_06213_b200 import _native as N

L = N.lib()
nb = 1 << 25
bounds, stream, rolls, words = bench.setup_c2(torch, B, 0, nb)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = [C.c_void_p(x.data_ptr()) for x in (bounds, stream.state, rolls, words)]
wsp = C.c_void_p(stream.workspace.data_ptr())


def run(phases, K=50):
    for _ in range(5):
        for ph in phases:
            L.br_roll_batches_phase(P[0], 2, nb, P[1], P[2], P[3], None, None, wsp, ph, sp)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        for ph in phases:
            L.br_roll_batches_phase(P[0], 2, nb, P[1], P[2], P[3], None, None, wsp, ph, sp)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K * 1e3


print("phase3 (main+fixup, PDL) us/step", run([3]))
print("phase1 only us/step", run([1]))
print("phase1 then phase2 us/step", run([1, 2]))
print("phase3 again", run([3]))
