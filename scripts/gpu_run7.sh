timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x -k "streamk or decode or tiny or ragged or onehot" > gpurun_out/t9.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/t9.log
python scripts/launch_floor.py 2>&1 | tail -4
python bench.py --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('value', d['value'], 'ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], d['clocks'])"
TM_PROFILE=1 python -m paper_2508_15601_b200.build > /dev/null && python scripts/trace_gemm.py 16 28672 4096 2>&1 | grep -E "per |timeline|   [a-z]"
