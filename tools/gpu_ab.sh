set -x
O=gpurun_out/ab
mkdir -p $O
for v in default match; do
  if [ $v = default ]; then unset SMX_LIB_PATH; else export SMX_LIB_PATH=paper_2512_09502_b200/_build/var_$v/libspikemesh_b200.so; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --model-ms 10 --prop-warmup-ms 1 > $O/bench_$v.json 2>&1
  python -c "import json; d=json.load(open('$O/bench_$v.json')); print('$v', d['ms_per_step'], d['phase_ms'])"
done
unset SMX_LIB_PATH
timeout 600 python tools/diag_host.py > $O/diag1.log 2>&1; head -12 $O/diag1.log
