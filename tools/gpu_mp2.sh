set -x
export PYTHONFAULTHANDLER=1
O=gpurun_out/mp2c
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider > $O/pytest_mp.log 2>&1
tail -15 $O/pytest_mp.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench2.json 2> $O/bench2.err
cat $O/bench2.json; tail -5 $O/bench2.err
SMX_PEER_EXCHANGE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 3 --warmup 2 > $O/bench2_nccl.json 2> $O/bench2_nccl.err
cat $O/bench2_nccl.json; tail -3 $O/bench2_nccl.err
