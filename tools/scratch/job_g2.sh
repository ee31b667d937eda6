#!/bin/bash
timeout 500 python -m pytest tests/test_gpu_crt.py tests/test_gpu_parity_timed.py -x -q > gpurun_out/g2_tests.txt 2>&1
tail -1 gpurun_out/g2_tests.txt
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:crt_gemm2 -c 6 python tools/prof_run.py --size 1024 --steps 1 2>&1 | grep -E "gpu__time|tensor_cycles" | head -12
bash tools/scratch/job_lib_ab.sh
