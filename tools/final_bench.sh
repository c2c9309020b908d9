for c in C1 C2 C3 C4 C5; do for v in plain deflate augment oblique orthogonal; do
  if [ "$c" = "C5" ] && [ "$v" != "deflate" ] && [ "$v" != "plain" ]; then continue; fi
  timeout 300 python bench.py --config $c --variant $v --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$v','none', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), d['roofline']['kernel'], d['roofline']['frac'])" || echo "$c $v FAILED"
done; done
for c in C1 C2 C3 C4; do for v in deflate oblique; do
  timeout 300 python bench.py --config $c --variant $v --precond ssor --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$v','ssor', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), d['roofline']['kernel'], d['roofline']['frac'])" || echo "$c $v ssor FAILED"
done; done
