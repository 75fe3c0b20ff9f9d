# bench lines of the small workloads with the per-step L2 flush (state < 2x L2)
mkdir -p gpurun_out
for w in c1 c2 c3; do
  python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>gpurun_out/l2_$w.err > gpurun_out/l2_$w.json
  python -c "import json;d=json.loads(open('gpurun_out/l2_$w.json').read().strip().splitlines()[-1]);print('$w',d['value'],d['e2e']['value'],d['roofline']['timing'],d['config']['l2'])"
done
