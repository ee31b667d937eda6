#!/bin/bash
# BASELINE configs[4] sweep (2^12 .. 2^30 px) on the late round-2 build, with the CPU column
timeout 3000 python tools/sweep.py --min 12 --max 30 --tc-max 30 --cpu > gpurun_out/sw3_sweep.jsonl 2> gpurun_out/sw3_sweep.err
tail -3 gpurun_out/sw3_sweep.jsonl | cut -c1-200
