cd $GRAFT_REPO_ROOT
O=gpurun_out/ab; rm -rf $O; mkdir -p $O
timeout 300 python tools/xdot_check.py > $O/xdot_check.log 2>&1; echo rc=$? >> $O/xdot_check.log
MCR_LIB=$PWD/paper_1210_6412_b200/libmcr_dbg.so timeout 600 python tools/xdot_check.py > $O/xdot_check_dbg.log 2>&1; echo rc=$? >> $O/xdot_check_dbg.log
for i in 1 2; do
for v in old new; do
  L=$PWD/paper_1210_6412_b200/libmcr_$v.so
  MCR_LIB=$L timeout 300 python tools/prof_xdot.py c2 2 > $O/prof_${v}_$i.log 2>&1
done; done
timeout 900 python -m pytest tests/test_gpu_dots.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
