set -x
O=gpurun_out/r2g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py -q -p no:cacheprovider > $O/pytest.log 2>&1
tail -3 $O/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print('default', d['ms_per_step'], d['phase_ms'])"
STACK=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 tools/trace_dist.py > $O/trace.log 2>&1
head -60 $O/trace.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_gen" -c 1 -o $O/gen_full python tools/prof_construct.py > $O/ncu_gen.log 2>&1
