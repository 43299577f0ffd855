O=gpurun_out/chunkprof
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"chunk_kernel|emit_kernel" --launch-skip 20 -c 2 -o $O/chunk python tools/prop_bench.py --runs 1 --ms 100 > $O/ncu.log 2>&1; tail -2 $O/ncu.log
