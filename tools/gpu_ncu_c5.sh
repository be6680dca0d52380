set -x
REPS=2 timeout 300 python tools/shuffle_time.py c5 default > gpurun_out/c5_time.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:shuffle_stage_kernel -s 1 -c 1 -o gpurun_out/ncu_r2_c5stage python tools/shuffle_time.py c5 default > gpurun_out/ncu_c5.log 2>&1
echo ncu=$?
