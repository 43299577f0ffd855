for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2978$N bench.py --gpus $N --steps 8 --warmup 3 > /tmp/g$N.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('/tmp/g$N.json') if l.startswith('{')][-1]); print('gpus', $N, d['ms_per_step'], d['phase_ms'], d['rtf'])"
done
