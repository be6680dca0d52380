timeout 900 ncu --set full --clock-control none --import-source on -k regex:shuffle_stage_kernel -s 1 -c 1 -o gpurun_out/ncu_stage_$1 python tools/shuffle_time.py c5 default > gpurun_out/ncu_stage_$1.log 2>&1
echo ncu=$?
