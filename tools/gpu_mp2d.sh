set -x
O=gpurun_out/mp2e
mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 tools/diag_host.py > $O/diag2.log 2>&1
grep -v "^\*\|OMP\|NCCL" $O/diag2.log | head -50
SMX_FUSED=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/diag_host.py > $O/diag2g.log 2>&1
grep -v "^\*\|OMP\|NCCL" $O/diag2g.log | head -50
