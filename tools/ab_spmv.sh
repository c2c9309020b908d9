# standalone SpMV kernels (graph path) per library: tools/ab_spmv.sh "<bench args>" lib...
A="$1"; shift
for rep in 1 2; do for lib in "$@"; do
  RG_NO_PERSIST=1 RG_LIB_PATH=$lib timeout 300 python bench.py $A --no-cpu-baseline --no-e2e --no-vs-plain 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$A', '$lib'.split('/')[-1], round(d['value']*1e3,4), {k: (v['launches'], round(v['ms']*1e3/max(v['launches'],1),1), v['GBps']) for k, v in d['kernels'].items() if k.startswith('spmv') or k.startswith('dcgs')})" || echo "$A $lib FAILED"
done; done
