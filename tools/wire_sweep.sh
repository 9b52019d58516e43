B=paper_2103_04930_b200/bin
for slots in 2 3; do
  $B/avec-server --devices 0 --slots $slots > gpurun_out/ws_srv.log 2>&1 &
  SP=$!
  for i in $(seq 120); do grep -q "^listening on" gpurun_out/ws_srv.log && break; sleep 1; done
  EP=$(grep "^listening on" gpurun_out/ws_srv.log | awk '{print $3}')
  for c in 1 2 4 8; do
    echo "slots=$slots clients=$c $(timeout 300 $B/avec-loadgen --endpoint $EP --clients $c --steps 25 --warmup 2 --batch 8)"
  done
  kill $SP; wait $SP
done
nproc
