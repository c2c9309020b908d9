for rep in 1 2; do for env in "RG_X=1" "RG_P_STREAM=1"; do for c in C2 C3; do
  env $env timeout 300 python bench.py --config $c --variant deflate --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$env', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), {k: round(v['ms'],2) for k, v in d['kernels'].items() if k.startswith('p_')})"
done; done; done
