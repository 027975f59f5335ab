timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_cpp.py -x -q > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -1
python scripts/ktime.py 4194304 16 3 | head -4
python scripts/ktime_cfg5.py 2>/dev/null | grep -E "wall|row_prep"
python scripts/ktime_rmat.py 18 2>&1 | grep -E "wall|row_prep"
