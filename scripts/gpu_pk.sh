mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pk.py -x -q --timeout 600 > gpurun_out/pk_tests.log 2>&1; echo "pk tests $?"; tail -4 gpurun_out/pk_tests.log
timeout 300 python scripts/prefill_perf.py > gpurun_out/pk_perf.log 2>&1; echo "pk perf $?"; cat gpurun_out/pk_perf.log
TM_NO_PK=1 timeout 300 python scripts/prefill_perf.py --ms 2048,8192 > gpurun_out/tiled_perf.log 2>&1; echo "tiled perf $?"; cat gpurun_out/tiled_perf.log
