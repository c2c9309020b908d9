# DK1 tile-outer vs chunk-outer: gpu tests, C4/C3 bench lines, cold ncu of the DK1 launches, A/B.
O=gpurun_out/${1:-dk1}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/summary.txt
for c in C4 C3; do
  x=""; [ $c = C3 ] && x="--no-persist"
  timeout 600 python bench.py --config $c $x --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-vs-plain > $O/bench_$c.json 2> $O/bench_$c.err
done
B="python bench.py --no-graph --no-cpu-baseline --no-e2e --no-vs-plain"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:k_dk1 -s 300 -c 1 -o $O/c4_dk1 $B --config C4 --steps 4 --warmup 3 > $O/c4_dk1.log 2>&1
timeout 900 $N -k regex:k_dk1 -s 100 -c 1 -o $O/c3_dk1 $B --config C3 --no-persist --steps 3 --warmup 3 > $O/c3_dk1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dk -c 400 --csv --log-file $O/c4_dk_all.csv $B --config C4 --steps 1 --warmup 2 > $O/c4_dk_all.log 2>&1
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.summary.txt 2>&1; done
make -j16 rg EXPERIMENTS=1 > $O/make_exp.log 2>&1
bash tools/ab.sh "--config C4 --steps 8 --warmup 3" "-" "RG_DK1_CHUNK_OUTER=1" >> $O/summary.txt 2>&1
bash tools/ab.sh "--config C3 --no-persist --steps 8 --warmup 3" "-" "RG_DK1_CHUNK_OUTER=1" >> $O/summary.txt 2>&1
cat $O/summary.txt
