python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/t11.log 2>&1; tail -3 gpurun_out/t11.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sweep --csv --log-file gpurun_out/launches_c5b.csv python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c5b.log 2>&1; tail -1 gpurun_out/ncu_c5b.log | cut -c1-100
