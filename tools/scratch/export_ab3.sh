timeout 600 python -m pytest tests/test_gpu_results.py -q -p no:faulthandler 2>&1 | tail -2
for r in 1 2; do
for ex in 2 0; do
  for w in c5 m1 c2 c1 c3; do MPMB_EXPORT=$ex timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"export=$ex $w\",'%.4g'%d[\"value\"],'%.4g'%d[\"e2e\"][\"value\"])"; done
done; done
