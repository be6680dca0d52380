# full GPU check: tests, smoke, bench (tag in $1)
t=${1:-x}
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/full_${t}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/full_${t}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full_${t}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/full_${t}_bench.json 2> gpurun_out/full_${t}_bench.err
tail -2 gpurun_out/full_${t}_pytest.log; cat gpurun_out/full_${t}_smoke.log | tail -1
