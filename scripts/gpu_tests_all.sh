mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/tall.log 2>&1; echo "tests exit $?"
tail -15 gpurun_out/tall.log
