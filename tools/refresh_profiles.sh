#!/bin/bash
# Full measurement pass on a GPU box (gpurun): parity tests, smoke, the C2 bench line and the
# reference arm, the other configurations, the C2 launch list and ncu captures. Outputs under
# gpurun_out/; copy the ones to keep into profiles/ (round-tagged).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
bash tools/gpu_round.sh
timeout 600 python bench.py --config c1 > gpurun_out/cfg_c1.json 2> gpurun_out/cfg_c1.err
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/cfg_c3.json 2> gpurun_out/cfg_c3.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 1 > gpurun_out/cfg_c5.json 2> gpurun_out/cfg_c5.err
timeout 600 python bench.py --config c5 --n 20000000 --steps 5 --warmup 2 > gpurun_out/cfg_c5_20m.json 2> gpurun_out/cfg_c5_20m.err
timeout 300 python tools/time_c4.py > gpurun_out/cfg_c4.json 2> gpurun_out/cfg_c4.err
echo refresh done
