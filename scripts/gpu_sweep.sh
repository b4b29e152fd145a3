# configs[4] cell sweep + configs[1]/[2] density-rule layer sweeps
mkdir -p gpurun_out
python -m paper_2603_18636_b200.build > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python scripts/sweep.py cells --out gpurun_out/sweep_cells.jsonl > gpurun_out/sweep_cells.log 2>&1; echo "cells rc=$?"; tail -55 gpurun_out/sweep_cells.log
timeout 900 python scripts/sweep.py layers --config wan1.3b_480p --layers 30 --out gpurun_out/sweep_layers_wan13b.jsonl > gpurun_out/sweep_layers_wan13b.log 2>&1; echo "layers13 rc=$?"; tail -2 gpurun_out/sweep_layers_wan13b.log
timeout 1500 python scripts/sweep.py layers --config wan14b_720p --layers 40 --out gpurun_out/sweep_layers_wan14b.jsonl > gpurun_out/sweep_layers_wan14b.log 2>&1; echo "layers14 rc=$?"; tail -2 gpurun_out/sweep_layers_wan14b.log
