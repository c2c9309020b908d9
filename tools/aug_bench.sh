for c in C1 C2 C3; do for env in "RG_NO_PERSIST=1" "RG_X=1"; do
  env $env timeout 300 python bench.py --config $c --variant augment --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c augment','$env', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), d['roofline']['kernel'], d['roofline']['frac'])"
done; done
