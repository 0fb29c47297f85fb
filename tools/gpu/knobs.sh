for v in "KCG_TILED=0" "KCG_TILED_FROM=1024" "KCG_TILED_FROM=256" "KCG_REGISTER=1" "KCG_DROPIN_CACHE=0"; do
  echo "== $v"
  env $v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hubs.py tests/test_gpu_dropin.py -x -q -m gpu -k "tiered or hub or dropin or flicker" 2>&1 | tail -1
done
