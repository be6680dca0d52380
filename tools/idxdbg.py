import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd()+'/oracle')
import paper_2408_06213_b200 as B, oracle as O
for n, na in ((4096, 40), (4096, 3000), (4096, 65536)):
    data = torch.arange(n, dtype=torch.int32, device='cuda').repeat(na)
    try:
        B.shuffle_many(data, n, 99); torch.cuda.synchronize()
        print(n, na, B.last_kernel(), 'ok', flush=True)
    except Exception as e:
        print(n, na, 'FAIL', e, flush=True); break
