timeout 1500 python -m pytest tests/test_gpu_rng.py tests/test_gpu_facade.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/prop_bench.py --ms 100 --runs 3
timeout 600 python bench.py --workload c2 --steps 3 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], d['rtf'])"
