python -m pytest tests/test_gpu.py -x -q -k "small or c3 or lengths or custom or lehmer or naive or chacha or dispatch" 2>&1 | tail -2
REPS=20 python tools/shuffle_time.py c3 default
BR_SMALL_QUAD=1 BR_SMQ_FLAGS=2 REPS=20 python tools/shuffle_time.py c3 default
bash tools/gpu_ncu.sh c3i c3 shuffle_small_idx REPS=1; python tools/ncu_stalls.py gpurun_out/ncu_c3i.ncu-rep | grep -v "max\|min\|sum\|cycles_active";  python tools/ncu_kern.py gpurun_out/ncu_c3i.ncu-rep; rm gpurun_out/*.ncu-rep
