set -x
O=gpurun_out/mp2f
mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/diag_host.py > $O/diag2.log 2>&1
grep -v "^\*\|OMP\|NCCL" $O/diag2.log | head -40
TIMELINE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 tools/trace_dist.py > $O/trace_fused.log 2>&1
grep -v "^\*\|OMP\|NCCL\|Warn\|warn" $O/trace_fused.log | head -80
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29564 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench2.json 2> $O/bench2.err
cat $O/bench2.json; tail -3 $O/bench2.err
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench1.json 2> $O/bench1.err
cat $O/bench1.json; tail -3 $O/bench1.err
