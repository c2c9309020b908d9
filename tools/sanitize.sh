# compute-sanitizer over every execution path (tools/sanitize_cases.py); logs in gpurun_out/$1.
# the hand-rolled grid barriers, flag-carrying reductions, mbarrier rings and
# neighbour epochs are what racecheck / synccheck check.
O=gpurun_out/${1:-san}
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  for c in persistent graph cgs2 ssor bsr; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_cases.py $c > $O/${tool}_$c.log 2>&1
    echo "$tool $c rc=$?" | tee -a $O/summary.txt
  done
done
