set -x
O=gpurun_out/trace4
mkdir -p $O
TIMELINE=1 STACK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 tools/trace_dist.py > $O/trace_fused.log 2>&1
grep "^  gpu\|^rank0" $O/trace_fused.log | head -60
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29564 bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench2.json 2> $O/bench2.err
cut -c1-260 $O/bench2.json; tail -3 $O/bench2.err
timeout 600 python bench.py --steps 5 --warmup 3 > $O/bench1.json 2> $O/bench1.err
cut -c1-260 $O/bench1.json; tail -3 $O/bench1.err
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_multiprocess.py -q -x -p no:cacheprovider 2>&1 | tail -5
