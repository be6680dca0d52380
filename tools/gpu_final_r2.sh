# round-2 closing evidence: tests, smoke, both bench arms, the torchrun form at N = 1, launch list
set -x
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/fin/pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/fin/bench.json 2> gpurun_out/fin/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/fin/bench_reference.json 2> gpurun_out/fin/ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/fin/bench_torchrun1.json 2> gpurun_out/fin/torchrun.err; echo torchrun=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/fin/launches_bench.log 2>&1; echo launches=$?
python tools/launches_md.py gpurun_out/fin/launches_bench.csv 'Launch list of `python bench.py --steps 2 --warmup 1` (round 2, final kernels)' > gpurun_out/fin/launches_bench.md
