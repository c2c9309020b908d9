for rep in 1 2; do
for e in NONE RG_NO_FUSE_C=1; do
  if [ "$e" = "NONE" ]; then python bench.py --config C4 --steps 6 --no-cpu-baseline --no-e2e --no-vs-plain > gpurun_out/ab_$e.json 2> gpurun_out/ab_$e.err;
  else env $e python bench.py --config C4 --steps 6 --no-cpu-baseline --no-e2e --no-vs-plain > gpurun_out/ab_$e.json 2> gpurun_out/ab_$e.err; fi
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$e.json').read().strip().splitlines()[-1]); print('$e', d['value'], {k:(v['launches'], round(v['ms']/6,3)) for k,v in d['kernels'].items() if k in ('cbuild','gram','spmv_plain')})" || tail -3 gpurun_out/ab_$e.err
done; done
