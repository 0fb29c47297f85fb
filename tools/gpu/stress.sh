for a in "2 4 20" "2 4 20 pv" "3 4 10" "3 5 5" "4 6 5 pv" "2 5 3" "5 4 3" "5 4 3 pv" "1 4 50 pv" "1 3 50 pv"; do timeout 900 python tools/stress_repeat.py $a 2>&1 | tail -1; done
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_parity.py -k tiered -q 2>&1 | tail -1; done
