python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2,LODIE1 '[{"PBG_ROWTMA": "0"}, {}]' > gpurun_out/tma_ab2.txt 2>&1; cat gpurun_out/tma_ab2.txt
python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/c5.json 2>&1; tail -1 gpurun_out/c5.json | cut -c1-400
python bench.py --steps 20 --warmup 5 > gpurun_out/c4.json 2>&1; tail -1 gpurun_out/c4.json
