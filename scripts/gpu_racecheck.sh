# racecheck: every variant with the push cluster reduction disabled, then the push case alone (bounded)
TM_DEFS="TM_CLUSTER_PUSH=0" python -m paper_2508_15601_b200.build > /dev/null
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_racecheck_nopush.log 2>&1; echo "racecheck(no push) $?"; tail -2 gpurun_out/sanitize_racecheck_nopush.log
python -m paper_2508_15601_b200.build --force > /dev/null
SAN_ONLY=0 timeout 240 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitize_racecheck_push.log 2>&1; echo "racecheck(push, case 0) $?"; tail -2 gpurun_out/sanitize_racecheck_push.log
