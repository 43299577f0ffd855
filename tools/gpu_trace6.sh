O=gpurun_out/trace6
mkdir -p $O
TIMELINE=1 STACK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29563 tools/trace_dist.py > $O/trace_fused.log 2>&1
grep "^  gpu\|^rank0\|^  cpu" $O/trace_fused.log | head -100
