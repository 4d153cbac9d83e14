#!/bin/bash
# A/B helper: build variant libs from "NAME -DFLAG=.. ..." specs, then bench each
# on one gpurun call.  Usage: variants/ab.sh WORKLOAD "A -DX=1" "B -DX=0" ...
set -u
WL=$1; shift
cd /root/repo/paper_2511_02136_b200
names=""
for v in "$@"; do
  set -- $v; name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false "$@" \
    -Xcompiler -fPIC,-O2 -shared -o /root/repo/variants/libmlob_$name.so \
    csrc/mlob_kernels.cu csrc/mlob_policy.cu csrc/mlob_lobster.cu csrc/mlob_ppo.cu csrc/mlob_runtime.cu csrc/mlob_store.cpp -lcublas 2>&1 | grep " error" &
  names="$names $name"
done
wait
cd /root/repo
cmd="for v in $names; do MLOB_LIB=variants/libmlob_\$v.so python bench.py --workload $WL --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c \"import json,sys; d=json.loads(sys.stdin.read()); print('\$v', d['value'], d['ms_per_step'])\"; done"
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "$cmd" 2>&1 | grep -v "sending\|GPU-minutes"
