for v in 512 362 256; do
echo "== KCG_TILED_FROM=$v"
KCG_TILED_FROM=$v timeout 900 python tools/prof_c5.py 5 total,pv 2>&1 | tail -2 | cut -c1-70
KCG_TILED_FROM=$v timeout 600 python tools/prof_count.py --config 2 --k 4 --reps 3 2>&1 | tail -1 | cut -c1-80
done
