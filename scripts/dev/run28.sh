python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_plan.py -x -q > gpurun_out/t28.log 2>&1; tail -3 gpurun_out/t28.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{}]' > gpurun_out/ab28.txt 2>&1; cat gpurun_out/ab28.txt
