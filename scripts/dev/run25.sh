python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_plan.py tests/test_gpu_scale.py -x -q > gpurun_out/t25.log 2>&1; tail -5 gpurun_out/t25.log
python scripts/dev/fuse_ab.py c3,c4 LODIE2 '[{"PBG_ROWLEAN": "0"}, {}, {"PBG_FLOWK": "2"}]' > gpurun_out/ab25.txt 2>&1; cat gpurun_out/ab25.txt
C=c3; TAG=r02c
python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_rowlean -s 3 -c 1 -o gpurun_out/${C}_full_$TAG python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${C}_$TAG.log 2>&1
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page raw --csv > gpurun_out/${C}_full_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${C}_row_${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${C}_row_${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/${C}_full_$TAG.ncu-rep
