# A/B of the working tree against HEAD on the GPU box: tools/ab_tree.sh <outdir> "<bench args>" ["<bench args>" ...]
# The working tree's diff against HEAD (tools/ab.patch — not under gpurun_out/, which does not travel — written with
# `git diff HEAD -- paper_1807_09467_b200 > tools/ab.patch`) is reversed in a copy of the tree,
# which is built as the "A" (old) arm; the tree itself is "B" (new).  Alternating runs, two rounds.
O=$1; shift
mkdir -p $O
rm -rf /tmp/abold && mkdir -p /tmp/abold && cp -r . /tmp/abold/ 2>/dev/null
(cd /tmp/abold && patch -R -p1 < tools/ab.patch > /dev/null && rm -rf build/rg && make -j16 rg > /dev/null 2>&1) || echo "old tree build failed" >> $O/ab.txt
make -j16 rg > /dev/null 2>&1
for rep in 1 2; do
  for a in "$@"; do
    for arm in old new; do
      d=.; [ $arm = old ] && d=/tmp/abold
      (cd $d && timeout 600 python bench.py $a --no-cpu-baseline --no-e2e --no-vs-plain 2>/dev/null | tail -1) > $O/tmp.json
      python -c "
import json,sys
d=json.loads(open('$O/tmp.json').read())
ks=d['kernels']
top=sorted(ks.items(),key=lambda kv:-kv[1]['ms'])[:6]
print('$arm', '$a', round(d['value']*1e3,4), sum(d['config']['iterations_timed']), ' '.join('%s=%.3f'%(k,v['ms']) for k,v in top))
" >> $O/ab.txt 2>&1 || echo "$arm $a FAILED" >> $O/ab.txt
    done
  done
done
cat $O/ab.txt
