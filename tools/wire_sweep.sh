B=paper_2103_04930_b200/bin
for slots in 2 3; do
  $B/avec-server --devices 0 --slots $slots > gpurun_out/ws_srv.log 2>&1 &
  SP=$!
  sleep 3
  EP=$(head -1 gpurun_out/ws_srv.log | awk '{print $3}')
  for c in 1 2 4 8; do
    echo "slots=$slots clients=$c $(timeout 300 $B/avec-loadgen --endpoint $EP --clients $c --steps 25 --warmup 2 --batch 8)"
  done
  kill $SP; wait $SP
done
nproc
