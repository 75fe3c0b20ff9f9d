timeout 600 python -m pytest tests/test_gpu_results.py -q -p no:faulthandler 2>&1 | tail -3
for r in 1 2; do
for cf in 1 0; do
  for w in c5 m1 c2 c1; do MPMB_CROSS_FRAME=$cf timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(\"cross=$cf $w\",'%.4g'%d[\"value\"],'%.4g'%d[\"e2e\"][\"value\"])"; done
done; done
timeout 1500 python -m pytest tests -q -m gpu -p no:faulthandler > gpurun_out/cross_tests.log 2>&1; tail -3 gpurun_out/cross_tests.log | cut -c1-300
