#!/bin/bash
# sanitizers over the chain v6 ring test (all six instantiations)
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/san7_memcheck.log \
    python -m pytest tests/test_gpu_crt.py -x -q -k chain6 > gpurun_out/san7_memcheck_pytest.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --log-file gpurun_out/san7_synccheck.log \
    python -m pytest tests/test_gpu_crt.py -x -q -k chain6 > gpurun_out/san7_synccheck_pytest.txt 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 --kernel-name kns=crt_chain6 \
    --log-file gpurun_out/san7_racecheck.log python -m pytest tests/test_gpu_crt.py -x -q -k chain6 > gpurun_out/san7_racecheck_pytest.txt 2>&1
for f in gpurun_out/san7_*.txt; do echo "== $f"; tail -n 1 $f; done
for f in gpurun_out/san7_*.log; do echo "== $f"; tail -n 1 $f; done
