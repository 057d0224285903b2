python -m pytest tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t48.log 2>&1; tail -3 gpurun_out/t48.log
python scripts/dev/slab_model.py 8 queued > gpurun_out/slab48.jsonl 2>gpurun_out/slab48.err; cat gpurun_out/slab48.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_slab" -c 100 --csv --log-file gpurun_out/slab_launches48_warm.csv python scripts/dev/slab_model.py 8 > gpurun_out/ncu48.log 2>&1
grep k_slab_interface gpurun_out/slab_launches48_warm.csv | tail -2 | cut -c1-60,300-
for R in 0 3; do
ncu --set full --clock-control none --import-source on -k regex:k_sweep_rowlean -s $((64+R)) -c 1 -o /tmp/rowlean_rank$R python scripts/dev/slab_model.py 8 > gpurun_out/ncu48_$R.log 2>&1
ncu -i /tmp/rowlean_rank$R.ncu-rep --page source --csv --print-source sass > gpurun_out/rowlean_rank${R}_sass.csv 2>/dev/null
done
ls -la gpurun_out/rowlean_rank*
