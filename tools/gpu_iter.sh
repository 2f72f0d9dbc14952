cd $GRAFT_REPO_ROOT
O=gpurun_out/r02q; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
MCR_GPU_DEVICES=0,0 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 1 > $O/c2_2shards.json 2> $O/c2_2shards.err
