timeout 1200 python -m pytest tests/test_gpu_crt.py tests/test_gpu_parity_timed.py tests/test_gpu_net.py tests/test_gpu_layers.py tests/test_gpu_streamed.py tests/test_gpu_dropin_cpp.py tests/test_gpu_stress.py -q -x > gpurun_out/m_tests.txt 2>&1; echo rc=$? >> gpurun_out/m_tests.txt
timeout 600 python bench.py --no-tc > gpurun_out/m_bench_sk.json 2> gpurun_out/m_bench_sk.err
timeout 600 python bench.py --net usk > gpurun_out/m_bench_usk.json 2> gpurun_out/m_bench_usk.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:crt_gemm2_kernel -c 1 -o gpurun_out/m_crt_gemm2_kernel python tools/prof_run.py --size 1024 --steps 1 > gpurun_out/m_ncu_gemm.log 2>&1
