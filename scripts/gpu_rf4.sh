mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rf.py -x -q --timeout 300 > gpurun_out/rf_tests.log 2>&1; echo "rf tests $?"; tail -5 gpurun_out/rf_tests.log
python scripts/rf_trace.py 1 28672 4096 2>&1 | head -12
timeout 300 python scripts/rf_perf.py --ms 1,8,16 --splits=-148,-296 2>&1
