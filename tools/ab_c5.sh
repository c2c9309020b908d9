# A/B library builds on C5 (SpMM): tools/ab_c5.sh lib...
for rep in 1 2; do for lib in "$@"; do
  RG_LIB_PATH=$lib python bench.py --config C5 --steps 3 --no-cpu-baseline --no-e2e --no-vs-plain > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$lib'.split('/')[-1], round(d['value']*1e3,4), {k:(v['launches'], round(v['ms']*1e3/max(1,v['launches']),1)) for k,v in d['kernels'].items() if k in ('spmv_plain','spmv_step')})" || tail -3 gpurun_out/ab.err
done; done
