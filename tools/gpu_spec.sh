set -x
O=gpurun_out/spec
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fused.py tests/test_gpu_multiprocess.py -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -15 $O/pytest.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N bench.py --gpus $N --steps 5 --warmup 3 > $O/c3_n$N.json 2> $O/c3_n$N.err
cut -c1-300 $O/c3_n$N.json; tail -3 $O/c3_n$N.err
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/c3_n1.json 2> $O/c3_n1.err
for f in $O/c3_n*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', d['n_gpus'], round(d['ms_per_step'],2), d.get('rtf'), d.get('phase_ms'))
"; done
