set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/v12_E.json 2> gpurun_out/v12_E.err
timeout 600 python bench.py --workload C > gpurun_out/v12_C.json 2> gpurun_out/v12_C.err
timeout 600 python bench.py --workload D > gpurun_out/v12_D.json 2> gpurun_out/v12_D.err
timeout 600 python bench.py --workload B > gpurun_out/v12_B.json 2> gpurun_out/v12_B.err
