mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity_r2.py -q --timeout 600 -k "prefill or mid or onehot or tiny or ragged or zero or ones or doubling or determin or partial or shard" > gpurun_out/mc_tests.log 2>&1; echo "tests $?"; tail -4 gpurun_out/mc_tests.log
timeout 300 python scripts/prefill_perf.py > gpurun_out/mc_perf.log 2>&1; echo "mc perf $?"; cat gpurun_out/mc_perf.log
TM_NO_MCAST=1 timeout 300 python scripts/prefill_perf.py --ms 2048,8192 > gpurun_out/nomc_perf.log 2>&1; echo "no-mc perf $?"; cat gpurun_out/nomc_perf.log
