import os, sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import torch, __graft_entry__
import paper_2408_06213_b200 as B
import oracle as O
os.environ["BR_SHUFFLE_KERNEL"] = "stage"
n, na, eb = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt = np.uint32 if eb == 4 else np.uint64
payload = np.arange(n * na, dtype=dt) * 3 + 1
dev = torch.from_numpy(payload.view(np.int32 if eb == 4 else np.int64).copy()).cuda()
_, w = B.shuffle_many(dev, n, 4321, array_index_base=17, return_words=True)
torch.cuda.synchronize()
print("kernel", B.last_kernel())
ref = payload.copy(); rw = O.shuffle_segmented(ref, n, 4321, array_index_base=17)
got = dev.cpu().numpy().view(dt)
bad = [a for a in range(na) if not np.array_equal(got[a*n:(a+1)*n], ref[a*n:(a+1)*n])]
print("bad arrays", len(bad), bad[:5], "words ok", np.array_equal(w.cpu().numpy().view(np.uint32), rw))
