python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; tail -c 2500 gpurun_out/bench_r01b.json
