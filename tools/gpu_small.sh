timeout 900 python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider -k "c3 or small or dispatch or KERNEL or forced or golden" 2>&1 | tail -4
REPS=10 timeout 300 python tools/shuffle_time.py c3 default 2>&1 | tail -1
BR_SMALL_ROWS=1 REPS=10 timeout 300 python tools/shuffle_time.py c3 default 2>&1 | tail -1
