python -m pytest tests -m gpu -x -q > gpurun_out/t42.log 2>&1; tail -5 gpurun_out/t42.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2 '[{}]' > gpurun_out/ab42.txt 2>&1; cat gpurun_out/ab42.txt
