set -x
O=gpurun_out/ab2
mkdir -p $O
for F in 1 0; do
SMX_FUSED=$F timeout 600 python bench.py --steps 5 --warmup 3 --cpu-sample-neurons 1000 > $O/b1_f$F.json 2> $O/b1_f$F.err
SMX_FUSED=$F timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$F bench.py --gpus 2 --steps 5 --warmup 3 > $O/b2_f$F.json 2> $O/b2_f$F.err
done
for f in $O/*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['rtf'], d['phase_ms'], d['roofline']['kernel_ms'])
"; done
