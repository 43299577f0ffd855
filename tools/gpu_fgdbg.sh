SMX_LIB_PATH=paper_2512_09502_b200/_build/var_fg3/libspikemesh_b200.so timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --model-ms 1 --prop-warmup-ms 1 2>&1 | tail -5
