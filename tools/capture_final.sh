# End-of-round evidence (round 2): default bench line, per-config lines with the CPU oracle baseline and
# plain GMRES beside them, ncu launch list of the default bench step, cold --set full captures of the
# dominant / verdict-named kernels, device timelines.  Outputs under gpurun_out/$1.
O=gpurun_out/${1:-final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 8 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config C4 --k 32 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C4_k32.json 2> $O/bench_C4_k32.err
for v in augment oblique orthogonal; do
  timeout 900 python bench.py --config C2 --variant $v --steps 12 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain > $O/bench_C2_$v.json 2> $O/bench_C2_$v.err
done
timeout 900 python bench.py --config C4 --precond ssor --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C4_ssor.json 2> $O/bench_C4_ssor.err
timeout 900 python bench.py --config C3 --precond ssor --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C3_ssor.json 2> $O/bench_C3_ssor.err
for c in C3 C4 C5; do timeout 600 python tools/trace.py $c deflate 2 > $O/trace_$c.txt 2>&1; done
B="python bench.py --no-graph --no-cpu-baseline --no-e2e --no-vs-plain"
N="ncu --set full --clock-control none --import-source on"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file $O/c5_launches.csv $B --steps 1 --warmup 3 > $O/c5_launch.log 2>&1
timeout 900 $N -k regex:k_spmv_bsr_tma -s 30 -c 1 -o $O/c5_spmv $B --steps 4 --warmup 3 > $O/c5_spmv.log 2>&1
timeout 900 $N -k regex:k_spmm_bsr_tma -s 8 -c 1 -o $O/c5_spmm $B --steps 10 --warmup 3 > $O/c5_spmm.log 2>&1
timeout 900 $N -k regex:k_dk1_tma -s 300 -c 1 -o $O/c4_dk1 $B --config C4 --steps 4 --warmup 3 > $O/c4_dk1.log 2>&1
timeout 900 $N -k regex:k_dk1_tma -s 300 -c 1 -o $O/c3_dk1 $B --config C3 --steps 4 --warmup 3 > $O/c3_dk1.log 2>&1
timeout 900 $N -k regex:k_ssor -s 200 -c 2 -o $O/c4_ssor $B --config C4 --precond ssor --steps 4 --warmup 3 > $O/c4_ssor.log 2>&1
timeout 900 $N -k regex:k_dk2_tma -s 300 -c 1 -o $O/c4_dk2 $B --config C4 --steps 4 --warmup 3 > $O/c4_dk2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dk -c 600 --csv --log-file $O/c4_dk_launches.csv $B --config C4 --steps 1 --warmup 3 > $O/c4_dk_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dk -c 600 --csv --log-file $O/c3_dk_launches.csv $B --config C3 --steps 1 --warmup 3 > $O/c3_dk_launch.log 2>&1
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.summary.txt 2>&1; done
ls -la $O
