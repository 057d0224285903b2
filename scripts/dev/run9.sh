python bench.py --steps 20 --warmup 5 > gpurun_out/c4_9.json 2>gpurun_out/c4_9.err; tail -1 gpurun_out/c4_9.json; tail -2 gpurun_out/c4_9.err
python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5_9.json 2>gpurun_out/c5_9.err; tail -1 gpurun_out/c5_9.json; tail -2 gpurun_out/c5_9.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5.log 2>&1; tail -2 gpurun_out/ncu_c5.log
