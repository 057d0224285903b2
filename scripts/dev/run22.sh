export PBG_FUSED12=0
C=c3; TAG=r02b
python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 9 -c 3 -o gpurun_out/${C}_full_$TAG python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${C}_$TAG.log 2>&1
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page raw --csv > gpurun_out/${C}_full_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_sweep_row > gpurun_out/${C}_row_${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_sweep_col > gpurun_out/${C}_col_${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source sass -k regex:k_sweep_col > gpurun_out/${C}_col_${TAG}_sass.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source sass -k regex:k_sweep_row > gpurun_out/${C}_row_${TAG}_sass.csv 2>/dev/null
rm -f gpurun_out/${C}_full_$TAG.ncu-rep
ls -la gpurun_out/*$TAG*
