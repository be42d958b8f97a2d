mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tp_symm.py tests/test_gpu_tp_classes.py -q -s --timeout 300 > gpurun_out/tp_symm_tests.log 2>&1; echo "tp tests $?"; tail -6 gpurun_out/tp_symm_tests.log
