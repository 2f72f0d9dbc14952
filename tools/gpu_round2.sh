#!/bin/bash
# Round-2 measurement pass on a GPU box (gpurun): parity tests, smoke, the C2 bench line (the
# reference-order dots) and the reference arm, C1 / C3 / C5-20M lines, a 2-shard line on one
# GPU (MCR_GPU_DEVICES=0,0), C4 times, the C2 launch list (host-issued loop so every launch
# is listed: ncu does not profile the body of a conditional graph node), full ncu captures of
# the Jacobi sweep and of k_xdot. Outputs under gpurun_out/$1 (default r02).
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/${1:-r02}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --config c1 > $O/cfg_c1.json 2> $O/cfg_c1.err
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 > $O/cfg_c3.json 2> $O/cfg_c3.err
MCR_GPU_DEVICES=0,0 timeout 600 python bench.py --gpus 2 --steps 3 --warmup 1 > $O/cfg_c2_2shards.json 2> $O/cfg_c2_2shards.err
timeout 600 python bench.py --config c5 --n 20000000 --steps 3 --warmup 1 > $O/cfg_c5_20m.json 2> $O/cfg_c5_20m.err
timeout 300 python tools/time_c4.py > $O/cfg_c4.json 2> $O/cfg_c4.err
MCR_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -c 8 -o $O/spmv_full -f python tools/prof_spmv.py --mv 2 --jit 3 --bit 0 > $O/ncu_spmv.log 2>&1
MCR_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_xdot --launch-skip 40 -c 4 -o $O/xdot_full -f python tools/prof_xdot.py c2 > $O/ncu_xdot.log 2>&1
echo done
