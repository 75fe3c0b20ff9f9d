# K8 with the affine term from the G2P phase (prea) vs base; then the GPU suite on prea
for r in 1 2; do
  bash tools/ab_engaged.sh c5 512 10
  bash tools/ab_engaged.sh m1 1 20
  bash tools/ab_engaged.sh c2 1 20
done
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
cp paper_2502_18437_b200/variants/lib_prea.so paper_2502_18437_b200/libmpm_b200.so
timeout 1200 python -m pytest tests -q -m gpu -x -p no:faulthandler 2>&1 | tail -3
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
