set -x
timeout 300 tools/_build/peaks > gpurun_out/peaks2.json 2> gpurun_out/peaks2.err; echo peaks rc=$?
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q > gpurun_out/shard.log 2>&1; echo shard rc=$?
tail -5 gpurun_out/shard.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench2.err
