for v in var_fg1/ var_fg3/ var_fg4/ var_fg5/; do
  echo "variant '$v'"
  SMX_LIB_PATH=paper_2512_09502_b200/_build/${v}libspikemesh_b200.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --model-ms 1 --prop-warmup-ms 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phase_ms'])"
done
