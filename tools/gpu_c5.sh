# C5: ncu capture of the stage kernel: key counters, stall reasons, per-source-line totals
bash tools/gpu_ncu.sh c5 c5 shuffle_stage_kernel REPS=1
python tools/ncu_kern.py gpurun_out/ncu_c5.ncu-rep > gpurun_out/ncu_c5_stage.txt
python tools/ncu_stalls.py gpurun_out/ncu_c5.ncu-rep | grep -v "max\|min\|sum\|cycles_active" >> gpurun_out/ncu_c5_stage.txt
python tools/ncu_lines.py gpurun_out/ncu_c5.ncu-rep 90 >> gpurun_out/ncu_c5_stage.txt
rm gpurun_out/*.ncu-rep
