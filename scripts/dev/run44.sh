ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_sweep|k_slab" -c 1200 --csv --log-file gpurun_out/slab_launches44.csv python scripts/dev/slab_model.py 8 > gpurun_out/ncu44.log 2>&1
tail -3 gpurun_out/ncu44.log
wc -l gpurun_out/slab_launches44.csv
