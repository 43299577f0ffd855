for F in 8 4 2; do
  SMX_PASS_A_FREE_SMS=$F timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2966$F bench.py --gpus 4 --steps 5 --warmup 3 > /tmp/f$F.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('/tmp/f$F.json') if l.startswith('{')][-1]); print('free', $F, d['ms_per_step'], d['phase_ms'])"
done
