python scripts/dev/fuse_ab.py c3,c4 LODIE2 '[{}]' > gpurun_out/ab65.txt 2>&1; cat gpurun_out/ab65.txt
