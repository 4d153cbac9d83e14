# final round measurements: bench lines for every workload + reference arm + launch list
set -x
python bench.py > gpurun_out/final_E.json 2> gpurun_out/final_E.err
python bench.py --workload C > gpurun_out/final_C.json 2> gpurun_out/final_C.err
python bench.py --workload B > gpurun_out/final_B.json 2> gpurun_out/final_B.err
python bench.py --workload D > gpurun_out/final_D.json 2> gpurun_out/final_D.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref_E.json 2> gpurun_out/final_ref_E.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_E.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1
