#!/bin/bash
# crt tests + one bench line, each under its own timeout
timeout 400 python -m pytest tests/test_gpu_crt.py tests/test_gpu_parity_timed.py -x -q > gpurun_out/q_tests.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/q.json 2>gpurun_out/q.err
python -c "
import json,sys; d=json.loads(open('gpurun_out/q.json').read().strip().splitlines()[-1]); r=d['roofline']; print('q', round(d['value']), {k: round(v,2) for k,v in r['ip1_breakdown_ms_per_step'].items()}, r['ip1_chain_fallbacks_per_launch'], d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value']))"
tail -2 gpurun_out/q_tests.txt
