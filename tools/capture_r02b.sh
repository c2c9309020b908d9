# Round-2 evidence, second pass: per-config bench lines (deflate + plain beside them), then the cold
# ncu captures of tools/capture_r02.sh (DK1/DK2/CSR at C4, DK1/SELL/persistent at C3, BSR SpMV/SpMM
# at C5 + the C5 launch list).  Outputs under gpurun_out/$1.
O=gpurun_out/${1:-cap2}
mkdir -p $O
for c in C1 C2 C3 C4; do
  timeout 600 python bench.py --config $c --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
bash tools/capture_r02.sh ${1:-cap2}
