# A/B two library builds on C4 (graph path), results to files: tools/ab_env_c4.sh libA libB
for rep in 1 2; do for lib in "$@"; do
  RG_LIB_PATH=$lib python bench.py --config C4 --steps 6 --no-cpu-baseline --no-e2e --no-vs-plain > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$lib'.split('/')[-1], round(d['value']*1e3,4), {k:(v['launches'], round(v['ms']*1e3/max(1,v['launches']),2), round(v['tail_ms']*1e3/max(1,v['launches']),2)) for k,v in d['kernels'].items() if k.startswith('dcgs')})" || tail -3 gpurun_out/ab.err
done; done
