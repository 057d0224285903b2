python -m pytest tests/test_gpu_slab.py -m gpu -x -q > gpurun_out/t47.log 2>&1; tail -3 gpurun_out/t47.log
python scripts/dev/slab_model.py 8 queued > gpurun_out/slab47.jsonl 2>gpurun_out/slab47.err; cat gpurun_out/slab47.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_slab|k_sweep" -c 1200 --csv --log-file gpurun_out/slab_launches47_warm.csv python scripts/dev/slab_model.py 8 > gpurun_out/ncu47.log 2>&1
grep k_slab_interface gpurun_out/slab_launches47_warm.csv | tail -2
for R in 0 3; do
ncu --set full --clock-control none --import-source on -k regex:k_sweep_rowlean -s $((64+R)) -c 1 -o /tmp/rowlean_rank$R python scripts/dev/slab_model.py 8 > gpurun_out/ncu47_$R.log 2>&1
ncu -i /tmp/rowlean_rank$R.ncu-rep --page raw --csv > gpurun_out/rowlean_rank${R}_raw.csv 2>/dev/null
ncu -i /tmp/rowlean_rank$R.ncu-rep --page source --csv --print-source cuda > gpurun_out/rowlean_rank${R}_src.csv 2>/dev/null
done
ls -la gpurun_out/rowlean_rank*
