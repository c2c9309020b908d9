O=gpurun_out/${1:-dk2}
mkdir -p $O
./tools/cutest/t_cols > $O/t_cols.txt 2>&1
make -j16 rg EXPERIMENTS=1 > $O/make_exp.log 2>&1
for c in C4; do
bash tools/ab.sh "--config $c --steps 8 --warmup 3" "-" "RG_DK1_CHUNK_OUTER=1" "RG_DK2_UY_LOADS=1" "RG_DK1_CHUNK_OUTER=1 RG_DK2_UY_LOADS=1" >> $O/summary.txt 2>&1
done
make rg > $O/make.log 2>&1
cat $O/summary.txt
