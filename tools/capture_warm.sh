# DK1 / DK2 / SpMV under ncu WITHOUT the L2 flush (--cache-control none): the state the graph leaves
# behind (u, y just written by the SpMV / update pass), next to the cold captures; plus the reference
# arm's duration at the default step count.  Outputs under gpurun_out/$1.
O=gpurun_out/${1:-warm}
mkdir -p $O
B="python bench.py --no-graph --no-cpu-baseline --no-e2e --no-vs-plain"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
for c in C3 C4; do
  timeout 900 ncu --metrics $M --cache-control none --clock-control none -k regex:"k_dk|k_spmv" -c 900 --csv --log-file $O/${c}_warm.csv $B --config $c --steps 1 --warmup 3 > $O/${c}_warm.log 2>&1
done
/usr/bin/time -v timeout 1800 python bench.py --impl reference > $O/reference_default.json 2> $O/reference_default.err
tail -3 $O/reference_default.err
