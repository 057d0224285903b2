python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{"PBG_ROWTMA": "0"}, {"PBG_ROWTMA": "0", "PBG_INPLACE": "1"}, {"PBG_INPLACE": "1"}]' > gpurun_out/ab8.txt 2>&1; cat gpurun_out/ab8.txt
