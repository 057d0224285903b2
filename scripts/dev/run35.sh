python scripts/dev/c5_axes.py > gpurun_out/c5axes35.txt 2>&1; cat gpurun_out/c5axes35.txt
python -m pytest tests/test_gpu_slab.py -x -q > gpurun_out/t35.log 2>&1; tail -3 gpurun_out/t35.log
for n in 8 4 2; do python scripts/dev/slab_model.py $n; done > gpurun_out/slab_model35.jsonl 2>&1; cat gpurun_out/slab_model35.jsonl
