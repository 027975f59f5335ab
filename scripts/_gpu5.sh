timeout 600 ncu --set full --import-source on --clock-control none -k k_tile --launch-count 1 -o gpurun_out/tile_src -f python scripts/probe_small.py 4194304 16 1 > gpurun_out/ncu_src.log 2>&1
tail -2 gpurun_out/ncu_src.log
