O=gpurun_out/hi12
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py -q -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --workload c4 --gpus 4 --steps 1 --warmup 1 > $O/c4_n4.json 2> $O/c4_n4.err
cut -c1-1200 $O/c4_n4.json; tail -3 $O/c4_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tests/mp_worker.py multi_area_2r 2>&1 | tail -2
