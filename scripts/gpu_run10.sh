timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x -k "streamk or decode or tiny or ragged or onehot" > gpurun_out/t13.log 2>&1; echo "tests exit $?"; tail -1 gpurun_out/t13.log
python scripts/launch_floor.py 2>&1 | tail -3
for d in 0 1851; do
TM_PROFILE=1 TM_DIAG=$d python -m paper_2508_15601_b200.build > /dev/null
echo "=== $d"
timeout 60 python scripts/trace_gemm.py 16 28672 4096 2>&1 | grep -E "per |   [a-z]"
done
python -m paper_2508_15601_b200.build --force > /dev/null
