# round-2 final: full GPU suite, smoke, bench (+ reference arm), bench launch list (our kernels), sanitizers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests_full.log 2>&1; echo "tests $?"; tail -3 gpurun_out/tests_full.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench $?"; tail -1 gpurun_out/bench_default.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref $?"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:w4a16 -c 300 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-prefill > gpurun_out/ncu_bench.log 2>&1; echo "launches $?"
# compute-sanitizer: one tool per gpurun call (B200_PROFILING.md), e.g.
#   gpurun -- 'compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_memcheck.log 2>&1'
