timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f13_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f13_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f13_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f13_smoke.log
for w in D E C B; do timeout 600 python bench.py --workload $w > gpurun_out/f13_$w.json 2> gpurun_out/f13_$w.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 -o gpurun_out/prof_D_f13 python bench.py --workload D --steps 3 --warmup 3 --no-cpu > gpurun_out/f13_ncu_D.log 2>&1
tail -n 2 gpurun_out/f13_gputests.log gpurun_out/f13_smoke.log
