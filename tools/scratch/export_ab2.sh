for r in 1 2; do
for ex in 2 1; do
  for w in m1 c2 c3; do MPMB_EXPORT=$ex timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"export=$ex $w\",'%.4g'%d[\"value\"],'%.4g'%d[\"e2e\"][\"value\"])"; done
done; done
