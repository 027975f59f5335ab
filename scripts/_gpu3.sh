timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_warp --launch-count 4 -o gpurun_out/new_src -f python scripts/probe_small.py 4194304 16 1 > gpurun_out/ncu_src.log 2>&1
tail -3 gpurun_out/ncu_src.log
