timeout 900 python -m pytest tests/test_gpu_fused.py -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --model-ms 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['phase_ms'], d['roofline']['frac'])"; done
