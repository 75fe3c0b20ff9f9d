# e2e A/B: frame-end export in the last G2P (MPMB_EXPORT=1) vs gather at fetch (0)
for r in 1 2; do
for ex in 1 0; do
  for w in c5 m1 c2 c1 c3; do MPMB_EXPORT=$ex timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"export=$ex $w\",'%.4g'%d[\"value\"],'%.4g'%d[\"e2e\"][\"value\"])"; done
done; done
