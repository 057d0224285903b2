python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{}, {"PBG_ROWLEAN_NW": "162"}, {"PBG_ROWLEAN_NW": "20"}, {"PBG_ROWLEAN_NW": "24"}]' > gpurun_out/ab27.txt 2>&1; cat gpurun_out/ab27.txt
