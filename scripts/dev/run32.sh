python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_plan.py tests/test_gpu_scale.py -x -q > gpurun_out/t32.log 2>&1; tail -3 gpurun_out/t32.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{}]' > gpurun_out/ab32.txt 2>&1; cat gpurun_out/ab32.txt
