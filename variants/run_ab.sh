#!/bin/bash
# A/B of prebuilt variant libs (variants/libmlob_NAME.so), alternating runs.
# usage: variants/run_ab.sh "WORKLOADS" NAME1 NAME2 ...   (e.g. "C E" BASE NEW)
WLS=$1; shift
names="$*"
cmd="for r in 1 2; do for wl in $WLS; do for v in $names; do MLOB_LIB=variants/libmlob_\$v.so timeout 300 python bench.py --workload \$wl --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c \"import json,sys; d=json.loads(sys.stdin.read()); print('\$wl', '\$v', '%.4g' % d['value'], '%.3f' % d['ms_per_step'])\"; done; done; done"
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "$cmd" 2>&1 | grep -v "sending\|GPU-minutes"
