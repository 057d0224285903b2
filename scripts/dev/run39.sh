python scripts/dev/c5_axes.py > gpurun_out/c5axes39.txt 2>&1; cat gpurun_out/c5axes39.txt
python -m pytest tests/test_gpu_batch.py tests/test_gpu_shapes.py -x -q > gpurun_out/t39.log 2>&1; tail -3 gpurun_out/t39.log
