nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/f_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f_gputest.txt 2>&1; echo rc=$? >> gpurun_out/f_gputest.txt
timeout 600 python bench.py > gpurun_out/f_bench_sk.json 2> gpurun_out/f_bench_sk.err
timeout 600 python bench.py --net u > gpurun_out/f_bench_u.json 2> gpurun_out/f_bench_u.err
timeout 600 python bench.py --net usk > gpurun_out/f_bench_usk.json 2> gpurun_out/f_bench_usk.err
timeout 600 python tools/crt_ab.py --min-k 4096 1024 > gpurun_out/f_crt_ab.txt 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_crt.py tests/test_gpu_net.py::test_full_sk_net_229 tests/test_gpu_layers.py tests/test_gpu_malis.py tests/test_gpu_streamed.py"
for tool in memcheck synccheck; do timeout 1200 $CS --tool $tool --print-limit 50 --log-file gpurun_out/f_san_$tool.log python -m pytest $T -q -p no:cacheprovider > gpurun_out/f_san_${tool}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/f_san_${tool}_pytest.txt; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tc > gpurun_out/f_ncu_bench.log 2>&1
