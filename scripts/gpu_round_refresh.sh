# full GPU suite, default bench line, ncu launch list / traffic / full capture (profiles refresh)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/tests_full.log 2>&1; echo "tests $?"; tail -2 gpurun_out/tests_full.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench $?"; tail -1 gpurun_out/bench_default.json
bash scripts/gpu_prof_r01.sh
