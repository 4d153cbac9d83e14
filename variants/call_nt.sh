# A/B only (no tests): VARS="A B" WLS="C E" bash variants/call_nt.sh
for r in 1 2; do for wl in ${WLS:-C E}; do for v in $VARS; do MLOB_LIB=variants/libmlob_$v.so timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl', '$v', '%.4g' % d['value'], '%.3f' % d['ms_per_step'])"; done; done; done
