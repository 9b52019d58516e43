#!/bin/bash
# Latency study of one pixel-major conv launch: rebuild libavec_cuda.so with
# -DAVEC_TRACE IN THIS CHECKOUT (run it in a scratch copy, e.g. on a gpurun
# box, never before committing product binaries) and print its CTA timeline.
set -e
make -B -j"$(nproc)" paper_2103_04930_b200/lib/libavec_cuda.so \
  NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DAVEC_TRACE" > /dev/null
for op in "$@"; do python tools/trace_op.py --config "${CONFIG:-c1}" --op "$op"; done
