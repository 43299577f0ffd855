set -x
O=gpurun_out/c2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_facade.py tests/test_gpu_memory.py -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -8 $O/pytest.log
timeout 900 python bench.py --workload c2 --steps 3 --warmup 1 > $O/c2_n1.json 2> $O/c2.err; cat $O/c2_n1.json; tail -3 $O/c2.err
