# device/e2e/wire throughput against execution slots per GPU
for r in 1 2; do
  for S in 2 3 4; do
    AVEC_SLOTS=$S python bench.py > gpurun_out/ab_b_slots${S}_${r}_c2.json 2>/dev/null
    AVEC_SLOTS=$S python bench.py --config c5 > gpurun_out/ab_b_slots${S}_${r}_c5.json 2>/dev/null
  done
done
