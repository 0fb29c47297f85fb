timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
python - <<'P'
import sys
sys.path.insert(0,'.')
from paper_2002_10047_b200 import gen, kcg
for cfg in (2,5):
    p = gen.CONFIGS[cfg]["rmat"]
    with kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"], permute=p["permute"]) as h:
        for _ in range(3):
            h.rank(gen.gpu_strategy(gen.CONFIGS[cfg]), gen.CONFIGS[cfg]["eps"], download=False)
            h.direct(download=False)
            tm = h.timings()
        print(cfg, 'rank_ms %.3f direct_ms %.3f' % (tm['rank_ms'], tm['direct_ms']))
P
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_warp -c 1 -o gpurun_out/c3k4_warp python tools/prof_count.py --config 3 --k 4 --reps 1 > gpurun_out/c3k4_warp.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_warp -c 1 -o gpurun_out/c4k6_warp python tools/prof_count.py --config 4 --k 6 --reps 1 > gpurun_out/c4k6_warp.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:count_warp -c 1 -o gpurun_out/c4k6pv_warp python tools/prof_count.py --config 4 --k 6 --reps 1 --pv > gpurun_out/c4k6pv_warp.log 2>&1; echo rc=$?
