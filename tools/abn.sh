# A/B/... of several librg.so builds: abn.sh CONFIG VARIANT lib1 lib2 ...; per-step CTA-0 phase times in us
C=$1; V=$2; shift 2
for rep in 1 2 3; do for lib in "$@"; do
  RG_LIB_PATH=$lib timeout 300 python bench.py --config $C --variant $V --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', '$lib'.split('/')[-1], round(d['value']*1e3,4), sum(d['config']['iterations_timed']), {k: round(v['ms']*1e3/max(v['launches'],1),2) for k, v in d['kernels'].items() if k.startswith('p_')})"
done; done
