# r02 profiles: launch list of the default bench, full captures of the c4 / c3 sweep kernels
TAG=${TAG:-r02a}
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
for C in c4 c3; do
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 9 -c 3 -o gpurun_out/${C}_full_$TAG python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${C}_$TAG.log 2>&1
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page raw --csv > gpurun_out/${C}_full_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${C}_full_$TAG.ncu-rep --page source --csv --print-source cuda,sass -k regex:k_sweep_row > gpurun_out/${C}_row_${TAG}_src.csv 2>/dev/null
rm -f gpurun_out/${C}_full_$TAG.ncu-rep
done
ls -la gpurun_out/*$TAG*
