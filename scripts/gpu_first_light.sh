set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
tail -5 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -x -k "pack or tiny" > gpurun_out/t1.log 2>&1; echo "t1 exit $?"
tail -30 gpurun_out/t1.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t2.log 2>&1; echo "t2 exit $?"
tail -60 gpurun_out/t2.log
