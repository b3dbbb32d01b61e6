for r in 1 2; do
for v in new old; do
  if [ $v = old ]; then export TMB_LIB=$PWD/paper_2405_04212_b200/libtmb200_old.so; else unset TMB_LIB; fi
  timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 3 > gpurun_out/abt_$v$r.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/abt_$v$r.json').read().strip().splitlines()[-1]); print('$v', d['value'])"
done; done
