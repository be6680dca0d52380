# round-2 evidence: launch list of the default bench, full captures of the C2 and C4 kernels
# (summaries written as text; the .ncu-rep files are deleted on the box)
set -x
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_bench.csv python bench.py --steps 2 --warmup 1 > gpurun_out/prof/launches_bench.log 2>&1
for spec in "c2roll c2 roll_fast_kernel" "c4idx c4 shuffle_idx_kernel"; do
  set -- $spec
  if [ $2 = c2 ]; then cmd="python bench.py --steps 1 --warmup 1 --no-secondary --no-cpu-baseline"; else cmd="python tools/shuffle_time.py $2 default"; fi
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o gpurun_out/prof/$1 $cmd > gpurun_out/prof/$1.log 2>&1
  python tools/ncu_kern.py gpurun_out/prof/$1.ncu-rep > gpurun_out/prof/$1.txt 2>&1
  python tools/ncu_hot.py gpurun_out/prof/$1.ncu-rep 25 >> gpurun_out/prof/$1.txt 2>&1
  rm -f gpurun_out/prof/$1.ncu-rep
done
