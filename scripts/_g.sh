./var_gather_bench > gpurun_out/gather_bench.txt 2>&1; cat gpurun_out/gather_bench.txt | tail -12
nproc; lscpu | grep "Model name"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json | cut -c1-400; tail -2 gpurun_out/bench_ref.err
