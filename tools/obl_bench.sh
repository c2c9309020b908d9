mkdir -p gpurun_out
for c in C1 C2 C3 C4; do for v in deflate oblique; do
  timeout 300 python bench.py --config $c --variant $v --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$v', d['value'], sum(d['config']['iterations_timed']), d['roofline']['frac'] if d.get('roofline') else None)" || echo "$c $v FAILED"
done; done
