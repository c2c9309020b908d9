mkdir -p gpurun_out
for c in C1 C2 C3 C4; do for pc in none ssor; do for v in deflate; do
  timeout 300 python bench.py --config $c --variant $v --precond $pc --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$pc','$v', d['value'], sum(d['config']['iterations_timed']), d['roofline']['kernel'], d['roofline']['frac'], {k: (v['ms'], v['GBps']) for k, v in d['kernels'].items() if k in ('ssor','spmv_step','dcgs_dots_ls','dcgs_update','persistent_solve')})" || echo "$c $pc $v FAILED"
done; done; done
