set -x
O=gpurun_out/trace1
mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 tools/trace_dist.py > $O/trace_fused.log 2>&1
grep -v "^\*\|OMP\|NCCL\|Warn\|warn" $O/trace_fused.log | head -30
SMX_FUSED=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29562 tools/trace_dist.py > $O/trace_general.log 2>&1
grep -v "^\*\|OMP\|NCCL\|Warn\|warn" $O/trace_general.log | head -30
