python -m pytest tests/test_stage.py -x -q 2>&1 | tail -3
python tools/c5_fill.py 148 256 296 2>&1 | grep arrays
