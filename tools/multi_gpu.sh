# Multi-GPU evidence on one box (run with gpurun --gpus N): bench.py at N ranks
# for C2 (weak) and C5 (strong), then C4: avec-server over all N GPUs driven by
# 2N native client sessions (affinity policy: one session stream per GPU slot).
N=${1:-4}
mkdir -p gpurun_out
B=paper_2103_04930_b200/bin
for n in 1 2 $N; do
  [ $n -gt $N ] && continue
  if [ $n -eq 1 ]; then
    python bench.py > gpurun_out/mg_c2_n1.json 2>gpurun_out/mg_c2_n1.err
    python bench.py --config c5 > gpurun_out/mg_c5_n1.json 2>gpurun_out/mg_c5_n1.err
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $n > gpurun_out/mg_c2_n$n.json 2>gpurun_out/mg_c2_n$n.err
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 \
      bench.py --gpus $n --config c5 > gpurun_out/mg_c5_n$n.json 2>gpurun_out/mg_c5_n$n.err
  fi
done
bash tools/c4_wire.sh $N > gpurun_out/mg_c4.txt 2>&1
