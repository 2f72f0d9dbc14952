cd $GRAFT_REPO_ROOT
O=gpurun_out/r02v; mkdir -p $O
timeout 300 python tools/xdot_check.py > $O/xdot_check.log 2>&1; echo rc=$? >> $O/xdot_check.log
MCR_LIB=$PWD/paper_1210_6412_b200/libmcr_dbg.so timeout 600 python tools/xdot_check.py > $O/xdot_check_dbg.log 2>&1; echo rc=$? >> $O/xdot_check_dbg.log
timeout 300 python tools/xdot_bench.py > $O/xb.log 2>&1
timeout 300 python tools/prof_xdot.py c2 3 > $O/prof.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dots.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
