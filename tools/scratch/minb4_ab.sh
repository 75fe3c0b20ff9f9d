for r in 1 2; do
  bash tools/ab_engaged.sh m1 1 20
  bash tools/ab_engaged.sh c5 512 10
  bash tools/ab_engaged.sh c2 1 20
done
