python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_plan.py tests/test_gpu_scale.py -x -q > gpurun_out/t23.log 2>&1; tail -5 gpurun_out/t23.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{"PBG_ROWLEAN": "0"}, {}, {"PBG_ROWLEAN_NW": "12"}, {"PBG_ROWLEAN_NW": "8"}]' > gpurun_out/ab23.txt 2>&1; cat gpurun_out/ab23.txt
