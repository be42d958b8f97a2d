timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/t10.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/t10.log
python scripts/launch_floor.py 2>&1 | tail -3
python bench.py --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', d['value'], 'ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], d['clocks'])"
for d in 0 15; do
  TM_PROFILE=1 TM_DIAG=$d python -m paper_2508_15601_b200.build > /dev/null
  echo "=== TM_DIAG=$d"
  python scripts/trace_gemm.py 16 28672 4096 2>&1 | grep -E "per |   [a-z]"
done
python -m paper_2508_15601_b200.build --force > /dev/null
