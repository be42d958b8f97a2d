mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x -k "streamk" > gpurun_out/t6.log 2>&1; echo "sk tests exit $?"
tail -5 gpurun_out/t6.log
timeout 300 python scripts/trace_gemm.py 16 28672 4096 2>&1 | head -30
timeout 600 python scripts/quick_perf.py --ms 1,16,64 > gpurun_out/perf3.log 2>&1; echo "perf exit $?"
cat gpurun_out/perf3.log
