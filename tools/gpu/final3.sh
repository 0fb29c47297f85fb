set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
tail -3 gpurun_out/gputest.log
timeout 3000 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 400 gpurun_out/bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-config5 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu rc=$?
python -c "import __graft_entry__ as g; g.smoke()"; echo smoke rc=$?
