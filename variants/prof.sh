# ncu full captures of the step kernel for configs C (register book) and D (deep book)
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 -o gpurun_out/prof_C_final python bench.py --workload C --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_C_final.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 4 -c 1 -o gpurun_out/prof_D_final python bench.py --workload D --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_D_final.log 2>&1
