# abx.sh "BENCH ARGS" lib1 lib2 ...: s/system of each build, 2 alternating repetitions
A=$1; shift
for rep in 1 2; do for lib in "$@"; do
  RG_LIB_PATH=$lib timeout 300 python bench.py $A --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$A', '$lib'.split('/')[-1], round(d['value']*1e3,4), sum(d['config']['iterations_timed']))"
done; done
