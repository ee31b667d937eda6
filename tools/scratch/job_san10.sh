#!/bin/bash
timeout 1800 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 --kernel-name kns=crt_chain6 --log-file gpurun_out/san10_racecheck.log python -m pytest tests/test_gpu_crt.py -x -q -k chain6 > gpurun_out/san10_racecheck_pytest.txt 2>&1
echo "$(tail -n 1 gpurun_out/san10_racecheck_pytest.txt) | $(tail -n 1 gpurun_out/san10_racecheck.log)"
