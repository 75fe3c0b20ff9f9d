set -e
mkdir -p gpurun_out
for r in 1 2; do
for lim in 0 256; do
  MPMB_TINY_MAX_GROUPS=$lim python bench.py --workload c1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('c1 tiny<=$lim',d['value'],d['e2e']['value'],d['kernel_ms'])"
done; done
python -m pytest tests -q -m gpu -x 2>&1 | tail -3
