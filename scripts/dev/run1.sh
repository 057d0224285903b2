python -m pytest tests/test_gpu_shapes.py tests/test_gpu_scale.py -x -q -k "not config4" > gpurun_out/t_shapes.log 2>&1; tail -5 gpurun_out/t_shapes.log
PBG_ROWTMA=0 python -m pytest tests/test_gpu_shapes.py -x -q > gpurun_out/t_shapes0.log 2>&1; tail -2 gpurun_out/t_shapes0.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{"PBG_ROWTMA": "0"}, {}, {"PBG_ROWTMA_NW": "16"}, {"PBG_ROWTMA_NW": "12"}, {"PBG_ROWTMA_NW": "8"}]' > gpurun_out/tma_ab.txt 2>&1; cat gpurun_out/tma_ab.txt
