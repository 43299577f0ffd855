set -x
O=gpurun_out/dbg
mkdir -p $O
export PYTHONFAULTHANDLER=1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tests/mp_worker.py balanced_2r_p2p > $O/w.log 2>&1
grep -v "^$" $O/w.log | tail -60
