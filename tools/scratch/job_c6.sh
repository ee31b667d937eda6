#!/bin/bash
# ncu --set full of the v6 chain kernel on the bench workload
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:crt_chain6 -c 1 -o gpurun_out/c6 python tools/prof_run.py --size 1024 --steps 1 > gpurun_out/c6_ncu.log 2>&1
ncu -i gpurun_out/c6.ncu-rep --page raw --csv > gpurun_out/c6_raw.csv 2>/dev/null
ncu -i gpurun_out/c6.ncu-rep --page details --csv > gpurun_out/c6_details.csv 2>/dev/null
ncu -i gpurun_out/c6.ncu-rep --page source --csv > gpurun_out/c6_source.csv 2>/dev/null
ls -la gpurun_out/c6*
