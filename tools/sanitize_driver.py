"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck).  Dev tool; checks the results against the oracle as well."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2408_06213_b200 as B  # noqa: E402


def check_many(n, na, eb, seed):
    dt = np.uint32 if eb == 4 else np.uint64
    payload = np.arange(n * na, dtype=dt)
    dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
    B.shuffle_many(dev, n, seed)
    kern = B.last_kernel()
    ref = payload.copy()
    O.shuffle_segmented(ref, n, seed)
    assert np.array_equal(dev.cpu().numpy().view(dt), ref), (n, eb, kern)
    return kern


kerns = set()
for n, na, eb in ((64, 300, 4), (100, 70, 8), (1000, 9, 4), (4096, 5, 4), (3000, 3, 8), (20000, 2, 8), (70000, 1, 4)):
    kerns.add(check_many(n, na, eb, 17))
for forced in ("idx", "warp", "hash"):  # the shared-memory group kernels on partial and full groups
    os.environ["BR_SHUFFLE_KERNEL"] = forced
    for n, na, eb in ((33, 40, 8), (1000, 9, 4), (4096, 4, 4), (5003, 3, 8)):
        kerns.add(check_many(n, na, eb, 23))
os.environ.pop("BR_SHUFFLE_KERNEL")
nb = 5000
bounds = O.gen_bounds(3, 2 * nb)
bounds[:200:2] = 0xFFFFFFFF
bounds[1:200:2] = 3006477107
src = O.pcg64(9)
rolls, words, _, _ = O.roll_batches(src, bounds, 2)
ds = B.DeviceStream(9)
r = B.roll_batches(ds, torch.from_numpy(bounds.view(np.int32)).cuda(), 2)
assert np.array_equal(r.rolls.cpu().numpy().view(np.uint32), rolls)
kerns.add(B.last_kernel())
r = B.roll_batches(ds, torch.from_numpy(O.gen_bounds(4, 3 * 999).view(np.int32)).cuda(), 3)
kerns.add(B.last_kernel())
s = B.Pcg64Source(5)
z = np.arange(10000, dtype=np.uint32)
B.shuffle_batched(s, z)
kerns.add(B.last_kernel())
torch.cuda.synchronize()
print("sanitize driver ok:", sorted(kerns))
