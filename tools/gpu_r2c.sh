set -x
O=gpurun_out/r2c
mkdir -p $O
timeout 600 python tools/diag_normal.py > $O/diag_normal.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x -p no:cacheprovider > $O/pytest_fused.log 2>&1
tail -3 $O/pytest_fused.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
cat $O/bench.json; tail -3 $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/construct_dram.csv python tools/prof_construct.py > $O/ncu_construct.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_gen|fb_scatter" -c 2 -o $O/fused_full python tools/prof_construct.py > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
