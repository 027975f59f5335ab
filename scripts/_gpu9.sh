timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python scripts/trident_logical.py 8 2 > gpurun_out/trident_p8_on4.json 2> gpurun_out/trident_p8.err; cat gpurun_out/trident_p8_on4.json; tail -3 gpurun_out/trident_p8.err
