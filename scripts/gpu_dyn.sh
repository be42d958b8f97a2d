mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rf.py -x -q --timeout 600 -k dynamic > gpurun_out/dyn_tests.log 2>&1; echo "dyn tests $?"; tail -5 gpurun_out/dyn_tests.log
timeout 300 python scripts/rf_perf.py --ms 1,8,16 > gpurun_out/dyn_perf.log 2>&1; echo "perf $?"; cat gpurun_out/dyn_perf.log
