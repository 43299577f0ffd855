O=gpurun_out/c4e
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_multiprocess.py tests/test_gpu_facade.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for N in 2 4; do timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N bench.py --workload c4 --gpus $N --steps 1 --warmup 1 > $O/c4_n$N.json 2> $O/c4_n$N.err; python -c "
import json; d=json.loads([l for l in open('$O/c4_n$N.json') if l.startswith('{')][-1]); print($N, d['ms_per_step'], d['facade_s'], d['phase_ms'])"; done
