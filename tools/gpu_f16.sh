SMX_PASS_A_FREE_SMS=16 timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider 2>&1 | tail -2
SMX_PASS_A_FREE_SMS=16 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29799 bench.py --gpus 4 --steps 5 --warmup 3 > /tmp/f16.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('/tmp/f16.json') if l.startswith('{')][-1]); print('free16 gpus4', d['ms_per_step'], d['phase_ms'], d['rtf'])"
