#!/bin/bash
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 --log-file gpurun_out/san9_memcheck.log python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san9_memcheck_pytest.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 --log-file gpurun_out/san9_synccheck.log python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san9_synccheck_pytest.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 --kernel-name kns=crt_chain6 --log-file gpurun_out/san9_racecheck.log python -m pytest tests/test_gpu_crt.py -x -q -k chain6 > gpurun_out/san9_racecheck_pytest.txt 2>&1
for f in gpurun_out/san9_*.txt; do echo "$f: $(tail -n 1 $f)"; done; for f in gpurun_out/san9_*.log; do echo "$f: $(tail -n 1 $f)"; done
