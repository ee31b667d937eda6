timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.txt 2>&1; echo rc=$? >> gpurun_out/v_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/v_gputest.txt 2>&1; echo rc=$? >> gpurun_out/v_gputest.txt
timeout 600 python bench.py > gpurun_out/v_bench_sk.json 2> gpurun_out/v_bench_sk.err
