timeout 900 python bench.py --workload c4-train --steps 2 > gpurun_out/c4.json 2> gpurun_out/c4.err; echo rc4=$?
timeout 900 python bench.py --workload c5-sparse --steps 2 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo rc5=$?
timeout 600 python bench.py --impl reference --workload c4-train --steps 1 > gpurun_out/c4r.json 2> gpurun_out/c4r.err; echo rc4r=$?
timeout 600 python bench.py --impl reference --workload c5-sparse --steps 1 > gpurun_out/c5r.json 2> gpurun_out/c5r.err; echo rc5r=$?
tail -3 gpurun_out/c4.err gpurun_out/c5.err
