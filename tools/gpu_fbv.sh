for v in var_fb1/ var_fb4/ var_fb5/ var_fb7/; do
  echo "variant '$v'"
  SMX_LIB_PATH=paper_2512_09502_b200/_build/${v}libspikemesh_b200.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --model-ms 1 --prop-warmup-ms 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phase_ms'])"
done
SMX_LIB_PATH=paper_2512_09502_b200/_build/var_fb7/libspikemesh_b200.so timeout 600 python -m pytest tests/test_gpu_fused.py -q -p no:cacheprovider 2>&1 | tail -1
