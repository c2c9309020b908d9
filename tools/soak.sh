# Soak run of the seeded GPU fuzz with other seed bases (each base = 60 new cases incl. n = 150,001):
#   tools/soak.sh <outfile> <base> [<base> ...]
O=$1; shift
for b in "$@"; do
  echo "== RG_FUZZ_SEED_BASE=$b" >> $O
  RG_FUZZ_SEED_BASE=$b timeout 1500 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_fuzz_bsr.py tests/test_gpu_fuzz_seq.py -q 2>&1 | tail -4 >> $O
done
cat $O
