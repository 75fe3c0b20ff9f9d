#!/bin/bash
# C1 / C2 / C3 bench lines (value, e2e, launches, per-class ms)
for w in c1 c2 c3; do
  python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$w', '%.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'], 'ms/step %.3f'%d['ms_per_step'], 'launches', d['gpu_launches'], d.get('kernel_ms', d.get('profile','')))"
done
