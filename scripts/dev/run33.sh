python scripts/dev/fuse_ab.py c3,c4 LODIE2 '[{}, {"PBG_ROWLEAN_NW": "20"}]' > gpurun_out/ab33.txt 2>&1; cat gpurun_out/ab33.txt
