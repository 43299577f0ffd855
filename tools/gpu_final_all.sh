# Final state check on a 4-GPU box: every GPU test (multi-process included),
# smoke, the default bench line and the reference arm.
O=gpurun_out/final_all
mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $O/pytest.log 2>&1; tail -5 $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; cut -c1-300 $O/bench.json; tail -3 $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; cut -c1-200 $O/bench_ref.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --steps 5 --warmup 3 > $O/bench4.json 2> $O/bench4.err; cut -c1-300 $O/bench4.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > $O/bench4_ref.json 2> $O/bench4_ref.err; cut -c1-200 $O/bench4_ref.json; tail -2 $O/bench4_ref.err
