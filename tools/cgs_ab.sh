O=gpurun_out/${1:-cgs}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cgs2 or orthogonalisation or dcgs2 or bsr" > $O/pytest_parity.log 2>&1; echo "parity rc=$?" >> $O/summary.txt
timeout 900 python -m pytest tests/test_gpu_fullparity.py -x -q -k "C5 or c5" > $O/pytest_full_c5.log 2>&1; echo "fullparity C5 rc=$?" >> $O/summary.txt
timeout 600 python bench.py --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
B="python bench.py --no-graph --no-cpu-baseline --no-e2e --no-vs-plain"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_tma -s 40 -c 3 -o $O/c5_cgs $B --config C5 --steps 6 --warmup 3 > $O/c5_cgs.log 2>&1
python tools/ncu_summary.py $O/c5_cgs.ncu-rep > $O/c5_cgs.summary.txt 2>&1
make -j16 rg EXPERIMENTS=1 > $O/make_exp.log 2>&1
bash tools/ab.sh "--config C5 --steps 12 --warmup 3" "-" "RG_NO_TMA_CGS=1" >> $O/summary.txt 2>&1
make rg > /dev/null 2>&1
cat $O/summary.txt
