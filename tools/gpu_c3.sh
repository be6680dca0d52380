# C3: parity subset, timing, and the ncu summary kept under profiles/
python -m pytest tests/test_gpu.py -x -q -k "small or c3 or lengths or custom or lehmer or naive or chacha or dispatch" 2>&1 | tail -2
REPS=30 python tools/shuffle_time.py c3 default
bash tools/gpu_ncu.sh c3i c3 shuffle_small_idx REPS=1
python tools/ncu_kern.py gpurun_out/ncu_c3i.ncu-rep > gpurun_out/ncu_c3_small_idx.txt
python tools/ncu_hot.py gpurun_out/ncu_c3i.ncu-rep 25 >> gpurun_out/ncu_c3_small_idx.txt
python tools/ncu_stalls.py gpurun_out/ncu_c3i.ncu-rep | grep -v "max\|min\|sum\|cycles_active" >> gpurun_out/ncu_c3_small_idx.txt
rm gpurun_out/*.ncu-rep
python bench.py --no-cpu-baseline > gpurun_out/bench_nocpu.log 2>&1
