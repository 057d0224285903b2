python -m pytest tests/test_gpu_plan.py tests/test_gpu_shapes.py -x -q > gpurun_out/t_plan.log 2>&1; tail -3 gpurun_out/t_plan.log
PBG_RFLOW=1 python -m pytest tests/test_gpu_shapes.py -x -q -k row_warp > gpurun_out/t_rflow.log 2>&1; tail -2 gpurun_out/t_rflow.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2 '[{"PBG_ROWTMA": "0"}, {}, {"PBG_RFLOW": "1"}, {"PBG_RFLOW": "1", "PBG_ROWTMA_NW": "16"}, {"PBG_ROWTMA_NW": "16"}]' > gpurun_out/rflow_ab.txt 2>&1; cat gpurun_out/rflow_ab.txt
