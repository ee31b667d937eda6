#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_net.py tests/test_gpu_parity_timed.py tests/test_gpu_streamed.py tests/test_gpu_train.py tests/test_gpu_multigpu.py -x -q > gpurun_out/q2_tests.txt 2>&1
tail -1 gpurun_out/q2_tests.txt
for net in sk u usk; do
timeout 300 python bench.py --net $net --steps 5 --warmup 3 > gpurun_out/q2_$net.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/q2_$net.json').read().strip().splitlines()[-1]); print('$net', round(d['value']), {k: round(v,2) for k,v in d['layer_ms_per_step'].items() if k in ('ip3','ip1','conv22')})"
done
