for c in "2 4" "2 5" "3 4" "4 6" "4 8" "5 4"; do set -- $c; timeout 1500 python tools/ncu_counts.py --config $1 --k $2 --out gpurun_out/ncu_c$1k$2.json; done
timeout 1500 python tools/ncu_counts.py --config 5 --k 4 --pv --out gpurun_out/ncu_c5k4pv.json
timeout 1500 python tools/ncu_counts.py --config 4 --k 6 --pv --out gpurun_out/ncu_c4k6pv.json
