mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_gemm.py tests/test_gpu_parity_r2.py -q --timeout 600 -k "wide or prefill or mid or ragged or onehot or ones or zero or determin" > gpurun_out/wide_tests.log 2>&1; echo "tests $?"; tail -4 gpurun_out/wide_tests.log
timeout 300 python scripts/prefill_perf.py > gpurun_out/wide_perf.log 2>&1; echo "wide perf $?"; cat gpurun_out/wide_perf.log
TM_NO_WIDE=1 timeout 300 python scripts/prefill_perf.py --ms 2048,8192 > gpurun_out/nowide_perf.log 2>&1; echo "tiled perf $?"; cat gpurun_out/nowide_perf.log
