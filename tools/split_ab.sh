#!/bin/bash
for w in c1 c2 c3 m1; do
  for sp in 0 7104; do
    MPMB_SPLIT_MAX_GROUPS=$sp timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/split_${w}_$sp.json 2>gpurun_out/split_${w}_$sp.err
    python -c "
import json; d=json.loads(open('gpurun_out/split_${w}_$sp.json').read().strip().splitlines()[-1]); print('$w split<=$sp', '%.3e'%d['value'], 'ms/step %.3f'%d['ms_per_step'], {k: round(v,4) for k,v in d['kernel_ms'].items()})" 2>&1 | tail -1
  done
done
MPMB_SPLIT_MAX_GROUPS=7104 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_exact.py tests/test_dd.py tests/test_gpu_scale.py -q -x -m gpu 2>&1 | tail -3
MPMB_SPLIT_MAX_GROUPS=7104 timeout 1200 python -m pytest tests/test_gpu_horizon.py -q -x -m gpu -k "c1 or c5 or pose" 2>&1 | tail -3
