timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x -k "streamk or decode or tiny or ragged or onehot" > gpurun_out/t8.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/t8.log
timeout 600 python scripts/quick_perf.py --ms 1,16,64 2>&1
TM_PROFILE=1 python -m paper_2508_15601_b200.build > /dev/null && python scripts/trace_gemm.py 16 28672 4096 2>&1 | grep -E "per |kernel end|event"
