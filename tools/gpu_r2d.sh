set -x
O=gpurun_out/r2d
mkdir -p $O
timeout 600 python tools/diag_normal.py > $O/diag_normal.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_rng.py -q -p no:cacheprovider > $O/pytest.log 2>&1
tail -3 $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
cat $O/bench.json; tail -3 $O/bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_gen" -c 1 -o $O/gen_full python tools/prof_construct.py > $O/ncu_gen.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fb_scatter" -c 1 -o $O/scatter_full python tools/prof_construct.py > $O/ncu_sc.log 2>&1
tail -2 $O/ncu_sc.log
