mkdir -p gpurun_out/r1f
B=paper_2512_09502_b200/_build
run() { echo "== $*"; env "$@" timeout 120 python tools/sortbench.py 1.125e9 100000 2>&1 | tail -2; }
run ITERS=5 X=1
run ITERS=5 SMX_SORT_ALIAS=8
run ITERS=5 SMX_SORT_ALIAS=8 SMX_SORT_ALIAS_MID=8
for v in a4 a5; do
run ITERS=5 SMX_LIB_PATH=$B/var_$v/libspikemesh_b200.so SMX_SORT_ALIAS=8
run ITERS=5 SMX_LIB_PATH=$B/var_$v/libspikemesh_b200.so SMX_SORT_ALIAS=8 SMX_SORT_ALIAS_MID=8
done
echo "== check small"
for v in a4; do SMX_LIB_PATH=$B/var_$v/libspikemesh_b200.so SMX_SORT_ALIAS=8 SMX_SORT_ALIAS_MID=8 timeout 300 python tools/sortbench.py 3e7 100000 2>&1 | tail -2; SMX_LIB_PATH=$B/var_$v/libspikemesh_b200.so SMX_SORT_ALIAS=8 SMX_SORT_ALIAS_MID=8 timeout 300 python tools/sortbench.py 3.3e7 1000000 2>&1 | tail -2; done
