python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_plan.py tests/test_gpu_scale.py -x -q > gpurun_out/t29.log 2>&1; tail -5 gpurun_out/t29.log
python scripts/dev/fuse_ab.py c3 LODIE2,LODIE1 '[{"PBG_FUSED01": "0"}, {}, {"PBG_FUSED01_TW": "1"}, {"PBG_FUSED01_TW": "4"}, {"PBG_FUSED01_TW":"1","PBG_FUSED01_LAG":"8"}]' > gpurun_out/ab29.txt 2>&1; cat gpurun_out/ab29.txt
python scripts/dev/fuse_ab.py c4 LODIE2 '[{"PBG_FUSED01": "0"}, {}, {"PBG_FUSED01_LAG": "1"}]' > gpurun_out/ab29b.txt 2>&1; cat gpurun_out/ab29b.txt
