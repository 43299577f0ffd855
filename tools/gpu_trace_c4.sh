set -x
O=gpurun_out/trace_c4
mkdir -p $O
C4=1 TIMELINE=1 STACK=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 tools/trace_dist.py > $O/trace.log 2>&1
grep "^rank0\|^  gap" $O/trace.log | head -30
grep "^  gpu" $O/trace.log | awk '$4+0 >= 0.3' | head -60
grep "^  cpu" $O/trace.log | head -150
