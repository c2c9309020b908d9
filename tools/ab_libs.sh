# A/B/... of library builds on the same box: tools/ab_libs.sh "<bench args>" lib1 lib2 ...  (ENV via RG_ABENV)
A="$1"; shift
for rep in 1 2; do for lib in "$@"; do
  env $RG_ABENV RG_LIB_PATH=$lib timeout 300 python bench.py $A --no-cpu-baseline --no-e2e --no-vs-plain 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$A', '$lib'.split('/')[-1], round(d['value']*1e3,4), sum(d['config']['iterations_timed']), d['roofline']['frac'], {k: round(v['ms']*1e3/max(v['launches'],1),2) for k, v in d['kernels'].items() if k.startswith('p_')})" || echo "$A $lib FAILED"
done; done
