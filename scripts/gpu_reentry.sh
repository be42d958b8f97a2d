# re-entry check: GPU suite, smoke, default bench line, per-shape quick perf (decode + prefill)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/tests_full.log 2>&1; echo "tests $?"; tail -3 gpurun_out/tests_full.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench $?"; tail -1 gpurun_out/bench_default.json | cut -c1-600
timeout 900 python scripts/quick_perf.py --ms 1,16,64,128,2048,4096,8192 > gpurun_out/quick_perf.log 2>&1; echo "qp $?"
