for rep in 1 2; do for env in "RG_X=1" "RG_SPMM_2CTA=1"; do
  env $env timeout 300 python bench.py --config C5 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5','$env', round(d['value']*1e3,4), d['config']['iterations_timed'], {k: (v['launches'], round(v['ms'],2), v['GBps']) for k, v in d['kernels'].items() if k == 'spmv_plain'})"
done; done
