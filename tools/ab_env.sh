# A/B one build under two values of an environment switch, interleaved:
#   bash tools/ab_env.sh AVEC_POOLFUSE 0 1   -> gpurun_out/ab_{lt,b}_<VAR><val>_<round>_<cfg>.json
VAR=$1; shift
for r in 1 2; do
  for v in "$@"; do
    tag=${VAR}${v}
    env $VAR=$v python tools/layer_table.py --config c2 --json gpurun_out/ab_lt_${tag}_${r}_c2.json > /dev/null 2>&1
    env $VAR=$v python tools/layer_table.py --config c5 --json gpurun_out/ab_lt_${tag}_${r}_c5.json > /dev/null 2>&1
    env $VAR=$v python bench.py > gpurun_out/ab_b_${tag}_${r}_c2.json 2>/dev/null
    env $VAR=$v python bench.py --config c5 > gpurun_out/ab_b_${tag}_${r}_c5.json 2>/dev/null
  done
done
