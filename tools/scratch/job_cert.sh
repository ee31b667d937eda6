timeout 900 python -m pytest tests/test_gpu_crt.py tests/test_gpu_parity_timed.py tests/test_gpu_net.py tests/test_gpu_streamed.py -q -x > gpurun_out/k_tests.txt 2>&1; echo rc=$? >> gpurun_out/k_tests.txt
timeout 600 python bench.py --no-tc > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:crt_certify2 -c 1 -o gpurun_out/k_certify python tools/prof_run.py --size 1024 --steps 1 > gpurun_out/k_ncu.log 2>&1
