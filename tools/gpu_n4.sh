set -x
O=gpurun_out/n4
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -q -p no:cacheprovider > $O/pytest_mp.log 2>&1; tail -5 $O/pytest_mp.log
for N in 1 2 4; do
  if [ $N = 1 ]; then
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/c3_n$N.json 2> $O/c3_n$N.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N --steps 5 --warmup 3 > $O/c3_n$N.json 2> $O/c3_n$N.err
  fi
  cut -c1-400 $O/c3_n$N.json; tail -3 $O/c3_n$N.err
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --workload c4 --gpus 4 --steps 1 --warmup 1 > $O/c4_n4.json 2> $O/c4_n4.err
cat $O/c4_n4.json; tail -5 $O/c4_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --strong --neurons 400000 --steps 3 --warmup 3 > $O/c3s_n4.json 2> $O/c3s_n4.err
cut -c1-400 $O/c3s_n4.json; tail -3 $O/c3s_n4.err
