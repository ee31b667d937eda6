#!/bin/bash
# sanitizers after the late changes (fractional CRT, packed narrow planes, narrow heads, xmax, gemm API cache)
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --log-file gpurun_out/san6_memcheck.log \
    python -m pytest tests/test_gpu_crt.py tests/test_gpu_layers.py "tests/test_gpu_net.py::test_narrow_head_matches_dmma" "tests/test_gpu_net.py::test_full_sk_net_229" -x -q > gpurun_out/san6_memcheck_pytest.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --log-file gpurun_out/san6_synccheck.log \
    python -m pytest tests/test_gpu_crt.py "tests/test_gpu_net.py::test_narrow_head_matches_dmma" -x -q > gpurun_out/san6_synccheck_pytest.txt 2>&1
for f in gpurun_out/san6_*.txt; do echo "== $f"; tail -n 1 $f; done
for f in gpurun_out/san6_*.log; do echo "== $f"; tail -n 2 $f; done
