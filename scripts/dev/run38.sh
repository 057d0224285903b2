python scripts/dev/c5_axes.py > gpurun_out/c5axes38.txt 2>&1; cat gpurun_out/c5axes38.txt
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{}]' > gpurun_out/ab38.txt 2>&1; cat gpurun_out/ab38.txt
python -m pytest tests -m gpu -x -q > gpurun_out/t38.log 2>&1; tail -3 gpurun_out/t38.log
