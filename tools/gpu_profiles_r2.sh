# Round-2 evidence on one B200: bench lines (ours, reference arm, C4, C5),
# the bench launch list, DRAM per kernel of one construction, --set full
# captures of pass A / pass B and of the propagation kernels.
set -x
O=gpurun_out/r2
mkdir -p $O
PART=${PART:-a}   # a: bench lines, launch list, DRAM, pass-A capture; b: pass-B and propagation captures
if [ "$PART" = a ]; then
timeout 900 python bench.py > $O/bench_line.json 2> $O/bench.err; cat $O/bench_line.json | cut -c1-400
timeout 900 python bench.py --impl reference > $O/bench_reference_line.json 2> $O/bench_ref.err; cat $O/bench_reference_line.json | cut -c1-300
timeout 900 python bench.py --workload c4 --steps 2 --warmup 1 > $O/c4_n1.json 2> $O/c4.err; cut -c1-300 $O/c4_n1.json
timeout 1500 python bench.py --workload c5 --steps 2 --warmup 1 > $O/c5_lines.json 2> $O/c5.err; cut -c1-200 $O/c5_lines.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; tail -2 $O/ncu_launch.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/construct_dram.csv python tools/prof_construct.py > $O/ncu_construct.log 2>&1; tail -2 $O/ncu_construct.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_gen" -c 1 -o $O/gen_full python tools/prof_construct.py > $O/ncu_gen.log 2>&1; tail -2 $O/ncu_gen.log
fi
if [ "$PART" = b ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fb_scatter" -c 1 -o $O/scatter_full python tools/prof_construct.py > $O/ncu_sc.log 2>&1; tail -2 $O/ncu_sc.log
# steady-state propagation kernels (the first launches of a run are skipped)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"deliver_step|lif_block" --launch-skip 200 -c 4 -o $O/prop_full python tools/prop_bench.py --runs 2 --ms 100 > $O/ncu_prop.log 2>&1; tail -2 $O/ncu_prop.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum --clock-control none -k regex:"deliver_step|lif_block" --launch-skip 200 -c 40 --csv --log-file $O/prop_metrics.csv python tools/prop_bench.py --runs 2 --ms 100 > $O/ncu_prop2.log 2>&1; tail -2 $O/ncu_prop2.log
timeout 900 python bench.py --workload c2 --steps 3 --warmup 1 > $O/c2_n1.json 2> $O/c2.err; cut -c1-300 $O/c2_n1.json
fi
ls -la $O
