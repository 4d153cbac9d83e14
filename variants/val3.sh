timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/v13_gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v13_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v13_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/v13_smoke.log
timeout 600 python bench.py --workload D > gpurun_out/v13_D.json 2> gpurun_out/v13_D.err
timeout 600 python bench.py > gpurun_out/v13_E.json 2> gpurun_out/v13_E.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 -o gpurun_out/prof_D_v13 python bench.py --workload D --steps 3 --warmup 3 --no-cpu > gpurun_out/v13_ncu_D.log 2>&1
tail -n 2 gpurun_out/v13_gputests.log gpurun_out/v13_smoke.log
