for rep in 1 2; do for lib in tools/ablib/librg_old.so paper_1807_09467_b200/lib/librg.so; do for c in C2 C4; do
  RG_LIB_PATH=$lib timeout 300 python bench.py --config $c --variant deflate --steps 10 --warmup 10 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c','$lib'.split('/')[-1], round(d['value']*1e3,4), sum(d['config']['iterations_timed']))"
done; done; done
