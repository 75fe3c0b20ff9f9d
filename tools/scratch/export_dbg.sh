for r in 1 2; do
for d in 0 1 2 3; do
  echo "dbg=$d"
  for w in c2 m1; do MPMB_EXPORT_DBG=$d timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"$w\",d[\"value\"],d[\"e2e\"][\"value\"], d[\"kernel_ms\"][\"g2p\"])"; done
done; done
