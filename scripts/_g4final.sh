# 4-GPU refresh: bench lines at N=2 and N=4, tile store timing on 4 GPUs
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "N=$N rc=$?"; tail -c 300 gpurun_out/bench_n$N.json
done
timeout 300 python scripts/tiles_bench.py 8 2 > gpurun_out/tiles4.txt 2>&1; tail -4 gpurun_out/tiles4.txt
timeout 300 python scripts/tiles_bench.py 4 4 >> gpurun_out/tiles4.txt 2>&1; tail -4 gpurun_out/tiles4.txt
