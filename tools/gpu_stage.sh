timeout 900 python -m pytest tests/test_stage.py -x -q -p no:cacheprovider 2>&1 | tail -15
REPS=5 timeout 300 python tools/shuffle_time.py c5 default 2>&1 | tail -2
