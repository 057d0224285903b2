python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{"PBG_ROWLEAN": "0"}, {}, {"PBG_FLOWSMALL": "0"}]' > gpurun_out/ab24.txt 2>&1; cat gpurun_out/ab24.txt
