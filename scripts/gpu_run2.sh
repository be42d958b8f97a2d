mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t3.log 2>&1; echo "tests exit $?"
tail -15 gpurun_out/t3.log
timeout 900 python scripts/quick_perf.py --sweep > gpurun_out/perf1.log 2>&1; echo "perf exit $?"
cat gpurun_out/perf1.log | grep -v sweep
grep sweep gpurun_out/perf1.log | head -80
