set -x
O=gpurun_out/c4d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -15 $O/pytest.log
timeout 900 python bench.py --workload c4 --steps 1 --warmup 1 > $O/c4_n1.json 2> $O/c4_n1.err
cat $O/c4_n1.json; tail -5 $O/c4_n1.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --workload c4 --gpus 2 --steps 1 --warmup 1 > $O/c4_n2.json 2> $O/c4_n2.err
cat $O/c4_n2.json; tail -5 $O/c4_n2.err
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/b1.json 2> $O/b1.err; cut -c1-300 $O/b1.json
