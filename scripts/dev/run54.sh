PBG_SLAB_BETA=0 ncu --set full --clock-control none --import-source on -k regex:k_slab_ends -s 40 -c 1 -o /tmp/ends python scripts/dev/slab_model.py 8 > gpurun_out/ncu54.log 2>&1
ncu -i /tmp/ends.ncu-rep --page raw --csv > gpurun_out/ends_raw.csv 2>/dev/null
ncu -i /tmp/ends.ncu-rep --page details > gpurun_out/ends_details.txt 2>/dev/null
ncu -i /tmp/ends.ncu-rep --page source --csv --print-source sass > gpurun_out/ends_sass.csv 2>/dev/null
ls -la gpurun_out/ends*
