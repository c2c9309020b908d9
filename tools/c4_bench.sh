for rep in 1 2; do for env in "RG_X=1" "RG_FORCE_PERSIST=1"; do
  env $env timeout 300 python bench.py --config C4 --variant deflate --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4','$env', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), d['roofline']['kernel'], d['roofline']['frac'], {k: round(v['ms'],2) for k, v in d['kernels'].items() if k.startswith('p_') or k in ('dcgs_dots_ls','dcgs_update','spmv_step')})" || echo "C4 $env FAILED"
done; done
