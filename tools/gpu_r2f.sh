set -x
O=gpurun_out/r2f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py -q -p no:cacheprovider > $O/pytest.log 2>&1
tail -3 $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print('default', d['ms_per_step'], d['phase_ms'])"
for lo in 8; do SMX_FUSED_LO=$lo timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --model-ms 1 --prop-warmup-ms 1 > $O/bench_lo$lo.json 2>&1; python -c "import json; d=json.load(open('$O/bench_lo$lo.json')); print('lo$lo', d['ms_per_step'], d['phase_ms'])"; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_gen" -c 1 -o $O/gen_full python tools/prof_construct.py > $O/ncu_gen.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fb_scatter" -c 1 -o $O/scatter_full python tools/prof_construct.py > $O/ncu_sc.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/construct_dram.csv python tools/prof_construct.py > $O/ncu_construct.log 2>&1
tail -2 $O/ncu_sc.log
