#!/bin/bash
# build variant libs from "NAME -DFLAG=.. ..." specs in parallel (variants/libmlob_NAME.so)
cd /root/repo/paper_2511_02136_b200
for v in "$@"; do
  set -- $v; name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false "$@" \
    -Xcompiler -fPIC,-O2,-pthread -shared -o /root/repo/variants/libmlob_$name.so \
    csrc/mlob_kernels.cu csrc/mlob_policy.cu csrc/mlob_lobster.cu csrc/mlob_ppo.cu csrc/mlob_runtime.cu csrc/mlob_store.cpp -lcublas 2>&1 | grep " error" &
done
wait
