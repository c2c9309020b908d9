for rep in 1 2; do for env in "RG_X=1" "RG_FORCE_PERSIST=1"; do
  env $env timeout 300 python bench.py --config C4 --variant deflate --precond ssor --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4 ssor','$env', round(d['value']*1e3,4), sum(d['config']['iterations_timed']))"
done; done
