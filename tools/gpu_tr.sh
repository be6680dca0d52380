python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_5_3.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_tr_20_5.json 2>/dev/null
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_tr_5_3.json 2>/dev/null
python - <<'PY'
import json
for f in ("b_5_3","b_tr_20_5","b_tr_5_3"):
    for line in open("gpurun_out/%s.json"%f):
        if line.startswith("{"):
            d=json.loads(line); s=d["secondary"]
            print(f, d["ms_per_step"], s["c3"]["ms_per_step"], s["c3"]["roofline"]["frac"], s["c4"]["ms_per_step"])
PY
