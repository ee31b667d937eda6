timeout 2400 python tools/sweep.py --min 12 --max 30 --tc-max 30 --cpu > gpurun_out/sw_sweep.jsonl 2> gpurun_out/sw_sweep.err
timeout 900 python tools/batch_bench.py > gpurun_out/sw_batch.jsonl 2> gpurun_out/sw_batch.err
