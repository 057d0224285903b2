# c4 scale parity, ncu source-level capture of the row sweeps (TMA and cp.async), reference arm on c4
python -m pytest tests/test_gpu_scale.py -x -q -k config4 > gpurun_out/t_c4.log 2>&1; tail -3 gpurun_out/t_c4.log
for T in 1 0; do
PBG_ROWTMA=$T ncu --set full --clock-control none --import-source on -k regex:k_sweep_row -s 3 -c 1 -o gpurun_out/c3_row_tma$T python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_row$T.log 2>&1
ncu -i gpurun_out/c3_row_tma$T.ncu-rep --page source --csv --print-source sass > gpurun_out/c3_row_tma${T}_sass.csv 2>/dev/null
ncu -i gpurun_out/c3_row_tma$T.ncu-rep --page raw --csv > gpurun_out/c3_row_tma${T}_raw.csv 2>/dev/null
rm -f gpurun_out/c3_row_tma$T.ncu-rep
done
( time python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/ref_c4.json 2> gpurun_out/ref_c4.err
tail -2 gpurun_out/ref_c4.json; tail -4 gpurun_out/ref_c4.err; free -g | head -2; nproc
