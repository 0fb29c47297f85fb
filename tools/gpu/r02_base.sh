set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
make -C tools/peaks >/dev/null 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
tail -3 gpurun_out/gputest.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 2000 gpurun_out/bench.err
for c in "2 4" "3 4" "2 5" "4 6" "5 4"; do set -- $c; timeout 600 python tools/prof_count.py --config $1 --k $2 --reps 2 2>&1 | tail -1 | cut -c1-160; done
timeout 600 tests/cpp/bin/api_bench 2 5 0
