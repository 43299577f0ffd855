O=gpurun_out/chain1
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_rng.py tests/test_gpu_parity.py tests/test_gpu_facade.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; tail -5 $O/pytest.log
timeout 300 python tools/prop_bench.py --ms 100 --runs 3
SMX_CHAIN_ONEPASS=0 timeout 300 python tools/prop_bench.py --ms 100 --runs 3
timeout 900 python bench.py --workload c2 --steps 3 --warmup 1 2>/dev/null | cut -c1-400
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', d['ms_per_step'], d['rtf'], d['propagation']['spikes'])"
