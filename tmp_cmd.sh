timeout 600 python -m pytest tests -m gpu -x -q -k "infer" 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/tr.json 2> gpurun_out/tr.err; echo rc=$?; head -c 300 gpurun_out/tr.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29532 bench.py --impl reference --gpus 1 --steps 1 --warmup 3 > gpurun_out/trr.json 2> gpurun_out/trr.err; echo rc=$?; head -c 300 gpurun_out/trr.json
