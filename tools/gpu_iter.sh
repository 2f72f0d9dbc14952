cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dots.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
for n in 500 2000 7647; do ./tools/xsbench_bin $n 2000; done > $O/xsbench.log 2>&1
timeout 300 python tools/time_c4.py > $O/c4.json 2> $O/c4.err
