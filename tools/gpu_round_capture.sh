# Round-end capture: default bench line (+ vs_plain, e2e, cpu_baseline), per-config deflate lines with
# the plain sequence beside them, ncu launch list of the default bench, one ncu --set full of the
# dominant kernel (k_solve_persistent, C2) and of k_cbuild.  Outputs under gpurun_out/$1.
set -x
O=gpurun_out/${1:-cap}
mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
for v in augment oblique orthogonal; do
  timeout 600 python bench.py --variant $v --steps 20 --no-cpu-baseline --no-e2e --no-vs-plain > $O/bench_C2_$v.json 2> $O/bench_C2_$v.err
done
timeout 600 python bench.py --config C4 --variant deflate --precond ssor --steps 8 --no-cpu-baseline --no-e2e > $O/bench_C4_ssor.json 2> $O/bench_C4_ssor.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve_persistent -s 1 -c 1 -o $O/persist python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-vs-plain > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cbuild -s 5 -c 1 -o $O/cbuild python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain > $O/ncu_cbuild.log 2>&1
ls -la $O
python tools/timeline.py C2 20 > $O/timeline_C2.txt 2>&1
python tools/timeline.py C2 20 plain > $O/timeline_C2_plain.txt 2>&1
