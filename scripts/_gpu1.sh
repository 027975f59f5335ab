set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_warp_numeric --launch-count 2 -o gpurun_out/num_src -f python scripts/probe_small.py 4194304 16 1 > gpurun_out/ncu_src.log 2>&1
tail -3 gpurun_out/ncu_src.log
