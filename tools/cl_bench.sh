for rep in 1 2; do for c in C2 C3; do for cs in 1 2 4 8; do
  RG_PERSIST_CLUSTER=$cs timeout 300 python bench.py --config $c --variant deflate --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','cs=$cs', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), d['roofline']['frac'], {k: round(v['ms'],2) for k, v in d['kernels'].items() if k.startswith('p_')})" || echo "$c $cs FAILED"
done; done; done
