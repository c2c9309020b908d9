for rep in 1 2; do for env in "RG_DK1_TILES=1" "RG_X=1"; do for c in C4 C3; do
  env $env RG_NO_PERSIST=1 timeout 300 python bench.py --config $c --variant deflate --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$env', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), {k: (round(v['ms'],2), v['GBps'], round(v['tail_ms'],2)) for k, v in d['kernels'].items() if k in ('dcgs_dots_ls',)})"
done; done; done
