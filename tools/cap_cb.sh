O=gpurun_out/${1:-cb}
mkdir -p $O
B="python bench.py --no-cpu-baseline --no-e2e --no-vs-plain"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:k_cbuild -s 5 -c 1 -o $O/c4_cbuild $B --config C4 --steps 6 --warmup 3 > $O/c4_cbuild.log 2>&1
timeout 900 $N -k regex:k_solve_persistent -s 5 -c 1 -o $O/c2_persist $B --config C2 --steps 4 --warmup 3 > $O/c2_persist.log 2>&1
timeout 900 $N -k regex:k_cbuild -s 5 -c 1 -o $O/c3_cbuild $B --config C3 --steps 6 --warmup 3 > $O/c3_cbuild.log 2>&1
for f in $O/*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.summary.txt 2>&1; done
