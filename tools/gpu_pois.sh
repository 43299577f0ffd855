for m in 64 128 256; do echo "min steps $m"; SMX_POIS_MIN_STEPS=$m timeout 300 python tools/prop_bench.py --ms 100 --runs 3; done
for m in 64 128 256; do echo "min steps $m (1000 ms)"; SMX_POIS_MIN_STEPS=$m timeout 300 python tools/prop_bench.py --ms 1000 --runs 2; done
