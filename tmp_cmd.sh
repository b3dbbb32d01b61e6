timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-secondary > gpurun_out/bench_fast.json 2> gpurun_out/bench_fast.err; tail -c 1500 gpurun_out/bench_fast.json
