# C4: avec-server over N GPUs, 2N/4N/8N concurrent native sessions (TCP loopback)
N=${1:-4}
mkdir -p gpurun_out
B=paper_2103_04930_b200/bin
DEV=$(seq -s, 0 $((N - 1)))
for pol in affinity split; do
  $B/avec-server --devices $DEV --slots 2 --policy $pol > gpurun_out/c4_srv_$pol.log 2>&1 &
  SP=$!
  for i in $(seq 180); do grep -q "^listening on" gpurun_out/c4_srv_$pol.log && break; sleep 1; done
  EP=$(grep "^listening on" gpurun_out/c4_srv_$pol.log | awk '{print $3}')
  for c in 8 $((2 * N)) $((4 * N)); do
    echo "policy=$pol gpus=$N clients=$c $(timeout 300 $B/avec-loadgen --endpoint $EP --clients $c --steps 30 --warmup 3 --batch 8)"
  done
  kill $SP; wait $SP
done
echo "host cores: $(nproc)"
