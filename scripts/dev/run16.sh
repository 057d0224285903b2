python -m pytest tests/test_gpu_shapes.py -x -q > gpurun_out/t16.log 2>&1; tail -1 gpurun_out/t16.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{}]' > gpurun_out/ab16.txt 2>&1; cat gpurun_out/ab16.txt
