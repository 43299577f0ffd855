for r in 1 2; do
for v in "" var_sl0/ var_sl16/ var_sl256/; do
  SMX_LIB_PATH=paper_2512_09502_b200/_build/${v}libspikemesh_b200.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --model-ms 1 --prop-warmup-ms 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), d['phase_ms'])"
done
done
