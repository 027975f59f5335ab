timeout 1500 python scripts/configs.py --configs 3 --rmat-scale 22 > gpurun_out/config3_s22.jsonl 2> gpurun_out/config3_s22.err; cat gpurun_out/config3_s22.jsonl; tail -3 gpurun_out/config3_s22.err
