python -m pytest tests/test_gpu_batch.py tests/test_gpu_plan.py tests/test_gpu_shapes.py -x -q > gpurun_out/t10.log 2>&1; tail -3 gpurun_out/t10.log
python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5_10.json 2>gpurun_out/c5_10.err; tail -1 gpurun_out/c5_10.json; tail -3 gpurun_out/c5_10.err
python bench.py --config c5 --steps 20 --warmup 3 --c5-streams --no-e2e --no-cpu-baseline > gpurun_out/c5s_10.json 2>&1; tail -1 gpurun_out/c5s_10.json | cut -c1-200
