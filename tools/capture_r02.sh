# Round-2 cold-cache ncu evidence for the kernels VERDICT r1 names (one GPU, one process at a time):
#   C4: k_dk1_tma, k_dk2_tma, k_spmv_csr (graph path, the bench's launch configuration)
#   C3: k_dk1_tma on the graph path (--no-persist) and the persistent solve (its production path)
#   C5: k_spmv_bsr_tma and k_spmm_bsr_tma at the bench's k (system 12, k_eff ~ 10)
# --no-graph: ncu cannot see kernels inside conditional CUDA graphs (same kernels, launched one by one).
O=gpurun_out/${1:-cap2}
mkdir -p $O
B="python bench.py --no-graph --no-cpu-baseline --no-e2e --no-vs-plain"
N="ncu --set full --clock-control none --import-source on"
timeout 900 $N -k regex:k_dk1_tma -s 300 -c 1 -o $O/c4_dk1 $B --config C4 --steps 4 --warmup 3 > $O/c4_dk1.log 2>&1
timeout 900 $N -k regex:k_dk2_tma -s 300 -c 1 -o $O/c4_dk2 $B --config C4 --steps 4 --warmup 3 > $O/c4_dk2.log 2>&1
timeout 900 $N -k regex:k_spmv_csr -s 300 -c 1 -o $O/c4_spmv $B --config C4 --steps 4 --warmup 3 > $O/c4_spmv.log 2>&1
timeout 900 $N -k regex:k_dk1_tma -s 100 -c 1 -o $O/c3_dk1 $B --config C3 --no-persist --steps 3 --warmup 3 > $O/c3_dk1.log 2>&1
timeout 900 $N -k regex:k_spmv_sell -s 100 -c 1 -o $O/c3_sell $B --config C3 --no-persist --steps 3 --warmup 3 > $O/c3_sell.log 2>&1
timeout 900 $N -k regex:k_solve_persistent -s 4 -c 1 -o $O/c3_persist python bench.py --no-cpu-baseline --no-e2e --no-vs-plain --config C3 --steps 3 --warmup 3 > $O/c3_persist.log 2>&1
timeout 900 $N -k regex:k_spmv_bsr_tma -s 60 -c 1 -o $O/c5_spmv $B --config C5 --steps 10 --warmup 3 > $O/c5_spmv.log 2>&1
timeout 900 $N -k regex:k_spmm_bsr_tma -s 10 -c 1 -o $O/c5_spmm $B --config C5 --steps 10 --warmup 3 > $O/c5_spmm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/c5_launches.csv $B --config C5 --steps 1 --warmup 3 > $O/c5_launch.log 2>&1
ls -la $O
