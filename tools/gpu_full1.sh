O=gpurun_out/full1
mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $O/pytest.log 2>&1; tail -6 $O/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
( time timeout 900 python bench.py ) > $O/bench.json 2> $O/bench.err; cut -c1-300 $O/bench.json; tail -4 $O/bench.err
( time timeout 900 python bench.py --impl reference ) > $O/bench_ref.json 2> $O/bench_ref.err; cut -c1-200 $O/bench_ref.json; tail -4 $O/bench_ref.err
