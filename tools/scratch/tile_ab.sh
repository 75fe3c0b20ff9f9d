# A/B of the P2G shared-memory tile (variants base / tile) and the parity suite on the tile build
set -u
for r in 1 2; do
  bash tools/ab_engaged.sh c5 512 10
  bash tools/ab_engaged.sh m1 1 20
  bash tools/ab_engaged.sh c2 1 20
done
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
cp paper_2502_18437_b200/variants/lib_tile.so paper_2502_18437_b200/libmpm_b200.so
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
