C=c3; TAG=r02d
python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep_rowlean -s 3 -c 1 -o gpurun_out/${C}_full_$TAG python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${C}_$TAG.log 2>&1
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page raw --csv > gpurun_out/${C}_full_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${C}_row_${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${C}_row_${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/${C}_full_$TAG.ncu-rep
