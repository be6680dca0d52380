"""A/B timing of shuffle_many on one config (dev tool; BR_LIB selects the library build)."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2408_06213_b200 as B

# argv[1]: a bench config name (c3/c4/c5) or n:arrays:elem_bytes
if ":" in sys.argv[1]:
    _n, _na, _eb = (int(x) for x in sys.argv[1].split(":"))
    cfg = {"n": _n, "arrays": _na, "eb": _eb, "seed": 7}
else:
    cfg = bench.SHUFFLE_CFG[sys.argv[1]]
n, na, eb = cfg["n"], cfg["arrays"], cfg["eb"]
data = B.pcg64_fill(cfg["seed"], n * na) if eb == 8 else torch.arange(n, dtype=torch.int32, device="cuda").repeat(na)
if eb == 8 and data.dtype != torch.int64:
    data = data.view(torch.int64)
for _ in range(3):
    B.shuffle_many(data, n, cfg["seed"])
torch.cuda.synchronize()
ts = []
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); B.shuffle_many(data, n, cfg["seed"]); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
print(sys.argv[1], os.environ.get("BR_LIB", "current"), "median ms", round(statistics.median(ts), 4), B.last_kernel())
