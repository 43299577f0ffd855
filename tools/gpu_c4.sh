set -x
O=gpurun_out/c4
mkdir -p $O
nvidia-smi --query-gpu=memory.total --format=csv
# 1 GPU: 4 areas (the per-GPU load of 32 areas on 8 GPUs, no remote exchange between GPUs)
timeout 900 python bench.py --workload c4 --steps 1 --warmup 1 > $O/c4_n1.json 2> $O/c4_n1.err
cat $O/c4_n1.json; tail -5 $O/c4_n1.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --workload c4 --gpus 2 --steps 1 --warmup 1 > $O/c4_n2.json 2> $O/c4_n2.err
cat $O/c4_n2.json; tail -5 $O/c4_n2.err
