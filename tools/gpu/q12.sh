timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_peel.py -x -q -m gpu 2>&1 | tail -2
python - <<'P'
import sys
sys.path.insert(0,'.')
from paper_2002_10047_b200 import gen, kcg
for cfg in (2,):
    p = gen.CONFIGS[cfg]["rmat"]
    with kcg.DeviceGraph.rmat(p["scale"], p["samples"], seed=p["seed"], permute=p["permute"]) as h:
        for _ in range(5):
            h.rank(gen.gpu_strategy(gen.CONFIGS[cfg]), gen.CONFIGS[cfg]["eps"], download=False)
            h.direct(download=False)
            tm = h.timings()
            print(cfg, 'rank_ms %.3f direct_ms %.3f' % (tm['rank_ms'], tm['direct_ms']))
P
