timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.txt 2>&1; echo rc=$? >> gpurun_out/u_smoke.txt
timeout 900 python -m pytest tests/test_gpu_parity_timed.py tests/test_gpu_net.py tests/test_gpu_crt.py tests/test_gpu_streamed.py -q -x > gpurun_out/u_tests.txt 2>&1; echo rc=$? >> gpurun_out/u_tests.txt
timeout 300 python bench.py --no-cpu --no-tc --steps 4 --warmup 3 > gpurun_out/u_b1.json 2>&1
timeout 300 python bench.py --no-cpu --no-tc --steps 4 --warmup 3 > gpurun_out/u_b2.json 2>&1
timeout 300 python bench.py --net u --steps 3 --warmup 3 > gpurun_out/u_u.json 2>&1
timeout 300 python bench.py --net usk --steps 3 --warmup 3 > gpurun_out/u_usk.json 2>&1
