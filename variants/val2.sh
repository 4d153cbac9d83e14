set -x
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v12_ref_E.json 2> gpurun_out/v12_ref_E.err
MLOB_BENCH_BACKEND=gloo MLOB_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --workload C > gpurun_out/v12_C_2rank_1gpu.json 2> gpurun_out/v12_C_2rank.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/v12_launches_E.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/v12_ncu_launch.log 2>&1
