python scripts/dev/c5_axes.py > gpurun_out/c5axes36.txt 2>&1; cat gpurun_out/c5axes36.txt
