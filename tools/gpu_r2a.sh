set -x
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2a/pytest.log 2>&1
tail -5 gpurun_out/r2a/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
cat gpurun_out/r2a/bench.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"lif_block|deliver_step" -c 4 -o gpurun_out/r2a/prop python tools/prop_bench.py --runs 1 --ms 20 > gpurun_out/r2a/ncu_prop.log 2>&1
tail -3 gpurun_out/r2a/ncu_prop.log
