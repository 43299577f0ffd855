set -x
O=gpurun_out/c5
mkdir -p $O
timeout 1500 python bench.py --workload c5 --steps 2 --warmup 1 > $O/c5.jsonl 2> $O/c5.err
cat $O/c5.jsonl; tail -5 $O/c5.err
