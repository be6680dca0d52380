# usage: gpu_ncu.sh <tag> <config> <kernel-regex> [env...]
tag=$1; cfg=$2; kre=$3; shift 3
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o gpurun_out/ncu_$tag python tools/shuffle_time.py $cfg default > gpurun_out/ncu_$tag.log 2>&1
echo ncu_$tag=$?
