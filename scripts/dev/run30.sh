python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_plan.py tests/test_gpu_scale.py -x -q > gpurun_out/t30.log 2>&1; tail -5 gpurun_out/t30.log
python scripts/dev/fuse_ab.py c3 LODIE2,LODIE1 '[{"PBG_COLWARP": "0"}, {}]' > gpurun_out/ab30.txt 2>&1; cat gpurun_out/ab30.txt
