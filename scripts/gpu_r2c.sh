mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_rf.py tests/test_gpu_tp_symm.py -q --timeout 600 > gpurun_out/tests_r2c.log 2>&1; echo "tests $?"; tail -3 gpurun_out/tests_r2c.log
