#!/bin/bash
# builds the committed (HEAD) kernel sources as variants/libmlob_BASE.so for A/B runs
set -e
rm -rf /root/repo/variants/old && mkdir -p /root/repo/variants/old/p/csrc /root/repo/variants/old/include
cd /root/repo
git show HEAD:include/mlob.h > variants/old/include/mlob.h
for f in $(git ls-tree --name-only HEAD paper_2511_02136_b200/csrc/); do git show HEAD:$f > variants/old/p/csrc/$(basename $f); done
cd variants/old/p
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false -Xcompiler -fPIC,-O2,-pthread -shared \
  -o /root/repo/variants/libmlob_BASE.so csrc/mlob_kernels.cu csrc/mlob_policy.cu csrc/mlob_lobster.cu csrc/mlob_ppo.cu \
  csrc/mlob_runtime.cu csrc/mlob_store.cpp -lcublas 2>&1 | grep " error" || true
