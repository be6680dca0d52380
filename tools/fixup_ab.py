import os, sys, ctypes as C, statistics
sys.path.insert(0, os.getcwd())
import torch
import __graft_entry__
__graft_entry__.build()
import paper_2408_06213_b200 as B
from paper_2408_06213_b200 import _native as N
import bench
first, nb = 0, bench.NB_C2
bounds, stream, rolls, words = bench.setup_c2(torch, B, first, nb)
L = N.lib()
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
ptrs = [C.c_void_p(x.data_ptr()) for x in (bounds, stream.state, rolls, words)]
wsp = C.c_void_p(stream.workspace.data_ptr())
def step():
    N.check(L.br_roll_batches_phase(ptrs[0], 2, nb, ptrs[1], ptrs[2], ptrs[3], None, None, wsp, 3, sp), "roll")
for mode in ["", "plain", "", "plain"]:
    if mode: os.environ["BR_ROLL_FIXUP"] = mode
    else: os.environ.pop("BR_ROLL_FIXUP", None)
    for _ in range(50): step()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200): step()
    b.record(); torch.cuda.synchronize()
    print(mode or "coop", a.elapsed_time(b) / 200 * 1000, "us/step")
