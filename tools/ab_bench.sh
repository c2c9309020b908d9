# A/B of two library builds on the same box: tools/ab_bench.sh CONFIG VARIANT [env...]
for rep in 1 2; do for lib in tools/ablib/librg_old.so paper_1807_09467_b200/lib/librg.so; do
  RG_LIB_PATH=$lib RG_NO_PERSIST=1 timeout 300 python bench.py --config $1 --variant $2 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1','$2','$lib'.split('/')[-1], round(d['value']*1e3,4), sum(d['config']['iterations_timed']), {k: (round(v['ms'],2), v['GBps']) for k, v in d['kernels'].items() if k in ('dcgs_dots_ls','dcgs_update','spmv_step')})"
done; done
