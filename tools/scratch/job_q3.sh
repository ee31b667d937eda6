#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_crt.py tests/test_gpu_parity_timed.py tests/test_gpu_net.py -x -q > gpurun_out/q3_tests.txt 2>&1
tail -1 gpurun_out/q3_tests.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:crt_xmax -c 3 python tools/prof_run.py --size 1024 --steps 1 2>&1 | grep -E "gpu__time" | head -3
