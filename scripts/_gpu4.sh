timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python scripts/ktime_rmat.py 18 2>&1 | tail -9
timeout 900 python scripts/configs.py --configs 1,2,4,5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; cat gpurun_out/configs.jsonl; tail -2 gpurun_out/configs.err
timeout 900 python scripts/configs.py --configs 3 --rmat-scale 18 >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err; tail -1 gpurun_out/configs.jsonl
