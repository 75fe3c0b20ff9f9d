# A/B of the K8 L2 discard (variants disc / nodisc), twice, then the GPU suite on the default build
for r in 1 2; do
  bash tools/ab_engaged.sh c5 512 10
  bash tools/ab_engaged.sh m1 1 20
  bash tools/ab_engaged.sh c2 1 20
done
python -m pytest tests -q -m gpu -x 2>&1 | tail -3
