O=gpurun_out/norm
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_facade.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; tail -4 $O/pytest.log
timeout 900 python bench.py --workload c2 --steps 3 --warmup 1 > $O/c2_n1.json 2> $O/c2.err; cut -c1-900 $O/c2_n1.json; tail -3 $O/c2.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/c3.json 2> $O/c3.err; python -c "
import json; d=json.loads(open('$O/c3.json').read().strip().splitlines()[-1]); print('c3', d['ms_per_step'], d['rtf'], d['propagation']['step_us'])"
