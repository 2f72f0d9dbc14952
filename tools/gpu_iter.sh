cd $GRAFT_REPO_ROOT
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dots.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 300 python tools/time_c4.py > $O/c4.json 2> $O/c4.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > $O/c1.json 2> $O/c1.err
