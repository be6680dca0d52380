# C4: ncu capture of the index kernel: key counters, stall reasons, per-source-line totals
python -m pytest tests/test_gpu.py -x -q -k "fixed_sequence" 2>&1 | tail -2
bash tools/gpu_ncu.sh c4 c4 shuffle_idx_kernel REPS=1
python tools/ncu_kern.py gpurun_out/ncu_c4.ncu-rep > gpurun_out/ncu_c4_idx.txt
python tools/ncu_stalls.py gpurun_out/ncu_c4.ncu-rep | grep -v "max\|min\|sum\|cycles_active" >> gpurun_out/ncu_c4_idx.txt
python tools/ncu_lines.py gpurun_out/ncu_c4.ncu-rep 70 >> gpurun_out/ncu_c4_idx.txt
python tools/ncu_hot.py gpurun_out/ncu_c4.ncu-rep 30 >> gpurun_out/ncu_c4_idx.txt
rm gpurun_out/*.ncu-rep
