O=gpurun_out/ft
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 1500 python bench.py --workload c5 --c5-rules fixed_total --steps 2 --warmup 1 > $O/c5.json 2> $O/c5.err; python -c "
import json
for l in open('$O/c5.json'):
    d=json.loads(l); print(d['config']['workload'], d.get('ms_per_step'), d.get('peak_bytes_per_synapse'), d['config'].get('store_path'), d.get('records_ok'))
"; tail -3 $O/c5.err
