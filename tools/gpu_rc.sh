for C in 6 4 3; do
  SMX_REPLAY_C=$C timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 297$C$C bench.py --gpus 4 --steps 8 --warmup 3 > /tmp/rc$C.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('/tmp/rc$C.json') if l.startswith('{')][-1]); print('c', $C, d['ms_per_step'], d['phase_ms'])"
done
