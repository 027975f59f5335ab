timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "trident or summa" > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
for cfg in "4 4,4" "4 4,1" "2 2,2"; do set -- $cfg
SPG_GRID=$2 SPG_SKIP_CPU=1 SPG_E2E_STEPS=1 SPG_BENCH_DEBUG=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $1 --steps 10 --warmup 3 > gpurun_out/b4.json 2> gpurun_out/b4.err; echo "grid $2 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/b4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['config'].get('grid'))"; grep "timeline" gpurun_out/b4.err | head -2 | cut -c1-250
done
