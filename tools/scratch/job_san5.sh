#!/bin/bash
# sanitizers over the CRT suite with certify v3 (TMA slabs) and chain v6 (swizzled weight rows)
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/san5_memcheck.log \
    python -m pytest tests/test_gpu_crt.py tests/test_gpu_parity_timed.py -x -q > gpurun_out/san5_memcheck_pytest.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --log-file gpurun_out/san5_synccheck.log \
    python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san5_synccheck_pytest.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 \
    --kernel-name kns=crt_chain6 --kernel-name kns=crt_certify3 \
    --log-file gpurun_out/san5_racecheck.log \
    python -m pytest tests/test_gpu_crt.py -x -q -k "chain6 or case0" > gpurun_out/san5_racecheck_pytest.txt 2>&1
for f in gpurun_out/san5_*.txt; do echo "== $f"; tail -n 1 $f; done
for f in gpurun_out/san5_*.log; do echo "== $f"; tail -n 2 $f; done
