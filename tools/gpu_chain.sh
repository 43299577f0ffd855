set -x
O=gpurun_out/chain
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; tail -8 $O/pytest.log
timeout 900 python bench.py --workload c2 --steps 3 --warmup 1 > $O/c2_n1.json 2> $O/c2.err; cut -c1-900 $O/c2_n1.json; tail -3 $O/c2.err
