set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_ -s 10 -c 11 -o gpurun_out/c2k4_${TAG:-x} python tools/prof_count.py --config 2 --k 4 --reps 2 > gpurun_out/c2k4_ncu.log 2>&1; echo ncu rc=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k concurrent 2>&1 | tail -30
