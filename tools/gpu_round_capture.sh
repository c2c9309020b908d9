set -x
mkdir -p gpurun_out/r1b
O=gpurun_out/r1b
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -1 $O/bench_default.json | head -c 300
for c in C1 C3 C4 C5; do
  timeout 400 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
RG_SKEW=10 timeout 200 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain > /dev/null 2> $O/skew_C2.err
RG_SKEW=10 timeout 200 python bench.py --config C3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain > /dev/null 2> $O/skew_C3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve_persistent -s 1 -c 1 -o $O/persist python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-vs-plain > $O/ncu_full.log 2>&1
ls -la $O
