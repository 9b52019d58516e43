B=paper_2103_04930_b200/bin
$B/avec-server --devices 0 --slots 2 > gpurun_out/wv_srv.log 2>&1 &
SP=$!
for i in $(seq 120); do grep -q "^listening on" gpurun_out/wv_srv.log && break; sleep 1; done
EP=$(grep "^listening on" gpurun_out/wv_srv.log | awk '{print $3}')
for rep in 1 2 3 4 5 6; do timeout 300 $B/avec-loadgen --endpoint $EP --clients 4 --steps 50 --warmup 2 --batch 8; done
kill $SP; wait $SP
nproc; cat /proc/loadavg
