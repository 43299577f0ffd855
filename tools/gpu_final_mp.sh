# Round-2 multi-GPU evidence (4 GPUs): multi-process parity, C3 weak and
# strong scaling, C4 at 2 and 4 GPUs, NCCL vs peer exchange.
O=gpurun_out/final_mp
mkdir -p $O
nvidia-smi topo -m > $O/topo.txt
timeout 900 python -m pytest tests/test_gpu_multiprocess.py tests/test_gpu_fused.py -q -p no:cacheprovider > $O/pytest_mp.log 2>&1; tail -3 $O/pytest_mp.log
run() {  # N out args...
  N=$1; out=$2; shift 2
  if [ $N = 1 ]; then timeout 900 python bench.py "$@" > $O/$out.json 2> $O/$out.err
  else timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N "$@" > $O/$out.json 2> $O/$out.err; fi
  python - "$O/$out.json" <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
    print(sys.argv[1].split("/")[-1], d["n_gpus"], round(d["ms_per_step"], 2), d.get("rtf"), d.get("phase_ms"), d["config"].get("store_path"))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
}
run 1 c3_n1 --steps 5 --warmup 3 --no-cpu-baseline
run 2 c3_n2 --steps 5 --warmup 3
run 4 c3_n4 --steps 5 --warmup 3
run 2 c3s_n2 --strong --steps 5 --warmup 3
run 4 c3s_n4 --strong --steps 5 --warmup 3
SMX_PEER_EXCHANGE=0 run 2 c3_n2_nccl --steps 3 --warmup 3
run 2 c4_n2 --workload c4 --steps 2 --warmup 1
run 4 c4_n4 --workload c4 --steps 2 --warmup 1
