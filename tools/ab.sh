# A/B two builds of libavec_cuda.so on one box: bash tools/ab.sh old new
L=paper_2103_04930_b200/lib/libavec_cuda.so
cp $L /tmp/cur.so
for r in 1 2; do
  for v in "$@"; do
    cp build/ab/$v.so $L
    python tools/layer_table.py --config c2 --json gpurun_out/ab_lt_${v}_${r}_c2.json > /dev/null 2>&1
    python tools/layer_table.py --config c5 --json gpurun_out/ab_lt_${v}_${r}_c5.json > /dev/null 2>&1
    python bench.py > gpurun_out/ab_b_${v}_${r}_c2.json 2>/dev/null
    python bench.py --config c5 > gpurun_out/ab_b_${v}_${r}_c5.json 2>/dev/null
  done
done
cp /tmp/cur.so $L
