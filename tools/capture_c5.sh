# C5 (bench default) profiler evidence: ncu launch list of one bench step, --set full of the Arnoldi BSR
# SpMV (k_spmv_bsr_tma) and of the C = A W SpMM (k_spmm_bsr_tma).  Kernels inside conditional CUDA graphs
# are invisible to ncu: --no-graph replays the same kernels one by one.  Outputs in gpurun_out/$1.
O=gpurun_out/${1:-c5cap}
mkdir -p $O
B="python bench.py --config C5 --no-graph --no-cpu-baseline --no-e2e --no-vs-plain"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv $B --steps 1 --warmup 3 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_bsr_tma -s 10 -c 1 -o $O/spmv $B --steps 1 --warmup 3 > $O/ncu_spmv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_bsr_tma -s 1 -c 1 -o $O/spmm $B --steps 1 --warmup 3 > $O/ncu_spmm.log 2>&1
ls -la $O
