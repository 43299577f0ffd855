set -x
O=gpurun_out/r2k
mkdir -p $O
timeout 600 python tools/diag_host.py > $O/diag_host.log 2>&1
cat $O/diag_host.log
SMX_FUSED=0 timeout 600 python tools/diag_host.py > $O/diag_host_general.log 2>&1
cat $O/diag_host_general.log
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_facade.py tests/test_gpu_parity.py tests/test_gpu_rng.py tests/test_gpu_memory.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > $O/pytest.log 2>&1
tail -3 $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print('default', d['ms_per_step'], d['phase_ms'], d['construction_wall_s'])"
