SKIP=7 tools/ncu_sum.sh c3k4_cta_small count_cta -- python tools/prof_count.py --config 3 --k 4 --reps 1
python - <<'P'
import sys
sys.path.insert(0,'.')
from paper_2002_10047_b200 import gen, kcg
g = gen.load_config_graph(3, cache=False)
spec = gen.CONFIGS[3]
with kcg.DeviceGraph.from_graph(g) as h:
    for _ in range(4):
        h.rank(gen.gpu_strategy(spec), spec["eps"], download=False)
        h.direct(download=False)
        tm = h.timings()
        print('c3 rank_ms %.3f direct_ms %.3f' % (tm['rank_ms'], tm['direct_ms']))
P
