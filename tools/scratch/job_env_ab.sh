#!/bin/bash
# same-box A/B of an environment switch: $1 = variable, then values (each value run 3 times, interleaved)
var=$1; shift
for rep in 1 2 3; do for v in "$@"; do
  env $var=$v timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$var=$v', round(d['value']), {k: round(v,2) for k,v in r['ip1_breakdown_ms_per_step'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/ab_log.txt
done; done
cat gpurun_out/ab_log.txt
