nvidia-smi --query-gpu=index,name --format=csv
SPG_HOST_PROF=1 SPG_BENCH_DEBUG=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; tail -c 2500 gpurun_out/bench_n2.json; grep "rank\|host ms" gpurun_out/bench_n2.err | tail -12
