O=gpurun_out/fbfull
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for N in 1 2 4; do
  if [ $N = 1 ]; then timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/c3_n$N.json 2>$O/c3_n$N.err
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2964$N bench.py --gpus $N --steps 5 --warmup 3 > $O/c3_n$N.json 2> $O/c3_n$N.err; fi
  python -c "import json; d=json.loads([l for l in open('$O/c3_n$N.json') if l.startswith('{')][-1]); print('c3', $N, d['ms_per_step'], d['rtf'], d['phase_ms'])"
done
for N in 2 4; do timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2965$N bench.py --workload c4 --gpus $N --steps 1 --warmup 1 > $O/c4_n$N.json 2> $O/c4_n$N.err; python -c "
import json; d=json.loads([l for l in open('$O/c4_n$N.json') if l.startswith('{')][-1]); print('c4', $N, d['ms_per_step'], d['phase_ms'])"; done
