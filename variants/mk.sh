#!/bin/bash
# rebuild libmlob.so and print ptxas stats of step_kernel<4> (dev helper)
make -s -C /root/repo/paper_2511_02136_b200 2>&1 | grep -E "error" ; ls -la --time-style=+%T /root/repo/paper_2511_02136_b200/libmlob.so | awk '{print "lib built", $6}'
cd /root/repo/paper_2511_02136_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo --fmad=false -Xptxas -v -c mlob_kernels.cu -o /tmp/k.o 2>&1 | grep -A3 "Compiling entry function '_ZN4mlob11step_kernelILi4" | grep -E "stack|registers"
