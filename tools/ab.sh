# A/B of bench settings: tools/ab.sh "<bench args>" "VAR=1" "-" ...  ("-": no extra environment).
# The library's environment knobs (csrc/knobs.cuh) are compiled out of product builds: build the A/B
# library first with `make rg EXPERIMENTS=1` (and rebuild with plain `make rg` afterwards).
A="$1"; shift
for rep in 1 2; do for e in "$@"; do
  ee=$e; [ "$e" = "-" ] && ee=""
  env $ee timeout 300 python bench.py $A --no-cpu-baseline --no-e2e --no-vs-plain 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$A', '$e', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), d['roofline']['kernel'], d['roofline']['frac'])" || echo "$A $e FAILED"
done; done
