cd $GRAFT_REPO_ROOT
O=gpurun_out/r02n; mkdir -p $O
MCR_LIB=$PWD/paper_1210_6412_b200/libmcr_tim.so MCR_XDOT_STATS=1 timeout 300 python tools/xdot_bench.py > $O/xb_tim.log 2>&1
timeout 300 python tools/xdot_bench.py > $O/xb.log 2>&1
