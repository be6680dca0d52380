timeout 900 python -m pytest tests/test_gpu.py -x -q -p no:cacheprovider -k "idx or c4 or dispatch or KERNEL or forced" 2>&1 | tail -3
REPS=10 timeout 300 python tools/shuffle_time.py c4 default 2>&1 | tail -1
