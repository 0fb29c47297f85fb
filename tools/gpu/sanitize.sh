timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -k "tiered" -x -q > gpurun_out/memcheck.log 2>&1; echo memcheck rc=$?
grep -c "Invalid\|ERROR SUMMARY" gpurun_out/memcheck.log; grep "ERROR SUMMARY\|passed\|failed" gpurun_out/memcheck.log | tail -3
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -k "tiered" -x -q > gpurun_out/racecheck.log 2>&1; echo racecheck rc=$?
grep "RACECHECK SUMMARY\|passed\|failed" gpurun_out/racecheck.log | tail -3
grep -B2 -A12 "Race reported\|hazard" gpurun_out/racecheck.log | head -80
