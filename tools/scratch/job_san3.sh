#!/bin/bash
# compute-sanitizer over the round-2 late kernels (chain v6 ring, activation prep v2, certify pairs)
timeout 300 python -m pytest tests/test_gpu_crt.py -x -q -k "chain6" > gpurun_out/san3_plain.txt 2>&1
for t in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 --log-file gpurun_out/san3_$t.log \
    python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san3_${t}_pytest.txt 2>&1
done
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --log-file gpurun_out/san3_racecheck.log \
  python -m pytest tests/test_gpu_crt.py -x -q -k "chain6" > gpurun_out/san3_racecheck_pytest.txt 2>&1
tail -2 gpurun_out/san3_*.txt; grep -c "Error\|Hazard" gpurun_out/san3_*.log; tail -3 gpurun_out/san3_*.log
