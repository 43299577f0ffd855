# fused path: tests, bench, per-launch DRAM bytes of one construction
set -x
O=gpurun_out/r2b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x -p no:cacheprovider > $O/pytest_fused.log 2>&1
tail -5 $O/pytest_fused.log
timeout 900 python -m pytest tests/test_gpu_rng.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_memory.py tests/test_gpu_facade.py -q -x -p no:cacheprovider > $O/pytest_parity.log 2>&1
tail -5 $O/pytest_parity.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
cat $O/bench.json; tail -3 $O/bench.err
SMX_FUSED=0 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_general.json 2> $O/bench_general.err
cat $O/bench_general.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/construct_dram.csv python tools/prof_construct.py > $O/ncu_construct.log 2>&1
tail -2 $O/ncu_construct.log
