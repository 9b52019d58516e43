#!/bin/bash
# Mixed-load soak of one avec-server on one GPU: concurrent pose-net sessions
# at C2 (8x656x368) and C1 (1x368x368) shapes, a tf32 pose net, BODY_25 and
# MockPose sessions, all at once for several rounds; every client must finish
# ok with an exact byte account, and the server's resident memory must not grow
# across rounds (plan caches and pinned pools are bounded).
set -u
S=paper_2103_04930_b200/bin/avec-server; L=paper_2103_04930_b200/bin/avec-loadgen
ROUNDS=${ROUNDS:-4}
$S --slots 2 --max-sessions 32 > /tmp/soak_srv.txt 2>&1 &
SP=$!
for i in $(seq 60); do grep -q listening /tmp/soak_srv.txt && break; sleep 1; done
EP=$(grep listening /tmp/soak_srv.txt | awk '{print $3}')
fail=0
for r in $(seq $ROUNDS); do
  pids=()
  $L --endpoint $EP --clients 3 --steps 40 --warmup 2 --batch 8 > /tmp/soak_a.json 2>&1 & pids+=($!)
  $L --endpoint $EP --clients 2 --steps 80 --warmup 2 --batch 1 --width 368 --height 368 > /tmp/soak_b.json 2>&1 & pids+=($!)
  $L --endpoint $EP --clients 1 --steps 20 --warmup 1 --batch 4 --input tf32 > /tmp/soak_c.json 2>&1 & pids+=($!)
  $L --endpoint $EP --clients 1 --steps 4 --warmup 1 --batch 4 --model posenet-body25 --width 1312 --height 736 > /tmp/soak_d.json 2>&1 & pids+=($!)
  $L --endpoint $EP --clients 2 --steps 60 --warmup 2 --batch 8 --model mockpose > /tmp/soak_e.json 2>&1 & pids+=($!)
  for p in "${pids[@]}"; do wait $p || fail=1; done
  for f in a b c d e; do
    ok=$(tail -1 /tmp/soak_$f.json | python -c 'import json,sys;d=json.loads(sys.stdin.read());print(d["ok"], d["fps"])' 2>/dev/null || echo "bad")
    echo "round $r client-set $f: $ok"
    case "$ok" in True*) ;; *) fail=1 ;; esac
  done
  echo "round $r server RSS $(ps -o rss= -p $SP) KB"
done
kill $SP; wait $SP 2>/dev/null
echo "soak fail=$fail"
exit $fail
