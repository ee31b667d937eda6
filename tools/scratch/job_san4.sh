#!/bin/bash
# sanitizers over the CRT suite after the chain-v6 barrier restructure; racecheck restricted to
# the new chain kernel, the activation prep and the certification
timeout 300 python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san4_plain.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --log-file gpurun_out/san4_synccheck.log \
    python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san4_synccheck_pytest.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 \
    --kernel-name kns=crt_chain6 --kernel-name kns=crt_x_kernel --kernel-name kns=crt_certify2 \
    --log-file gpurun_out/san4_racecheck.log \
    python -m pytest tests/test_gpu_crt.py -x -q -k "chain6 or case0" > gpurun_out/san4_racecheck_pytest.txt 2>&1
for f in gpurun_out/san4_*.txt; do echo "== $f"; tail -n 2 $f; done
for f in gpurun_out/san4_*.log; do echo "== $f"; tail -n 3 $f; done
