#!/bin/bash
for net in u usk; do timeout 300 python bench.py --net $net --steps 5 --warmup 3 --no-cpu --no-tc 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$net', round(d['value']))"; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 --log-file gpurun_out/san8_memcheck.log python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san8_memcheck_pytest.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 --log-file gpurun_out/san8_synccheck.log python -m pytest tests/test_gpu_crt.py -x -q > gpurun_out/san8_synccheck_pytest.txt 2>&1
for f in gpurun_out/san8_*.txt; do echo "$f: $(tail -n 1 $f)"; done; for f in gpurun_out/san8_*.log; do echo "$f: $(tail -n 1 $f)"; done
