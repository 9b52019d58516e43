# One-GPU evidence refresh (round 1): bench lines, reference arm, layer tables,
# ncu launch list and --set full captures of the main kernels, C3/wire sweeps.
set -x
mkdir -p gpurun_out/prof
O=gpurun_out/prof
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c5 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --impl reference > $O/ref_c2.json 2> /dev/null
python bench.py --impl reference --config c5 > $O/ref_c5.json 2> /dev/null
python tools/layer_table.py --config c2 --json $O/layers_c2.json > $O/layers_c2.txt 2>&1
python tools/layer_table.py --config c5 --json $O/layers_c5.json > $O/layers_c5.txt 2>&1
python tools/memcpy_sweep.py > $O/memcpy_sweep.json 2> $O/memcpy.err
bash tools/wire_sweep.sh > $O/wire_sweep.txt 2>&1
# launch list of the bench command (serialised, cold caches: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 > $O/ncu_launches.log 2>&1
# full captures: 7x7 swap-AB, the CTA-pair pixel-major conv, the fused head,
# the fused conv1_1+conv1_2+pool1 (and the unfused conv1_1 it replaces)
python tools/profile_forward.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 2 -c 1 -o $O/conv7x7 python tools/profile_forward.py > $O/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_pm -s 3 -c 1 -o $O/conv_pm_pair python tools/profile_forward.py > $O/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_head -s 1 -c 1 -o $O/conv_head python tools/profile_forward.py > $O/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv12 -c 1 -o $O/conv12 python tools/profile_forward.py > $O/ncu4.log 2>&1
AVEC_CONV12=0 ncu --set full --clock-control none --import-source on -k regex:conv_first -c 1 -o $O/conv_first python tools/profile_forward.py > $O/ncu5.log 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt
# BODY_25 stage head on CTA pairs (C5 shape)
python tools/profile_forward.py --family openpose_body25 --width 1312 --height 736 --batch 32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_head2 -s 2 -c 1 -o $O/conv_head2 \
    python tools/profile_forward.py --family openpose_body25 --width 1312 --height 736 --batch 32 > $O/ncu6.log 2>&1
# BODY_25 96-channel dense-block conv (C5, the 12th pixel-major launch): MMA issue-bound before the
# per-tap descriptors
ncu --set full --clock-control none --import-source on -k regex:conv_pm -s 11 -c 1 -o $O/conv_pm96 \
    python tools/profile_forward.py --family openpose_body25 --width 1312 --height 736 --batch 32 > $O/ncu7.log 2>&1
