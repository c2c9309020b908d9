for c in C2 C3; do for env in "RG_X=1"; do
  env $env timeout 300 python bench.py --config $c --variant deflate --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$env', round(d['value']*1e3,4), 'e2e', d['e2e']['value'], sum(d['config']['iterations_timed']), d['roofline']['frac'], {k: round(v['ms'],2) for k, v in d['kernels'].items() if k.startswith('p_')})" || echo "$c $env FAILED"
done; done
