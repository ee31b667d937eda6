timeout 900 python -m pytest tests/test_gpu_malis.py tests/test_gpu_streamed.py tests/test_gpu_dropin_cpp.py -q > gpurun_out/j5_tests.txt 2>&1; echo rc=$? >> gpurun_out/j5_tests.txt
timeout 600 python tools/malis_bench.py > gpurun_out/j5_malis_bench.json 2> gpurun_out/j5_malis_bench.err
timeout 600 python tools/malis_bench.py --patch 32 --batch 4736 > gpurun_out/j5_malis_bench32.json 2>> gpurun_out/j5_malis_bench.err
