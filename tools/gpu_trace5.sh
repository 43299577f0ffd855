O=gpurun_out/trace5
mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29561 tools/trace_dist.py > $O/trace_fused.log 2>&1
grep -v "^\*\|OMP\|NCCL\|Warn\|warn" $O/trace_fused.log | head -60
timeout 600 python tools/diag_host.py > $O/diag.log 2>&1; tail -40 $O/diag.log
