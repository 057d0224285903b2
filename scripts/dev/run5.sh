python -m pytest tests -m gpu -x -q > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 python scripts/dev/sanitize_small.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log; tail -4 gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --target-processes all --print-limit 50 python scripts/dev/sanitize_small.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log; tail -4 gpurun_out/san_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --target-processes all --print-limit 50 python scripts/dev/sanitize_small.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.log; tail -4 gpurun_out/san_synccheck.log
PBG_ROWTMA=0 ncu --set full --clock-control none --import-source on -k regex:k_sweep_row -s 3 -c 1 -o gpurun_out/c3_rw python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_rw.log 2>&1
ncu -i gpurun_out/c3_rw.ncu-rep --page source --csv --print-source cuda > gpurun_out/c3_rw_cuda.csv 2>/dev/null
ls -la gpurun_out/c3_rw*
