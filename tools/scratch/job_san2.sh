CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_crt.py tests/test_gpu_net.py::test_full_sk_net_229 tests/test_gpu_layers.py tests/test_gpu_malis.py tests/test_gpu_streamed.py"
for tool in memcheck synccheck; do timeout 1500 $CS --tool $tool --print-limit 50 --log-file gpurun_out/s2_san_$tool.log python -m pytest $T -q -p no:cacheprovider > gpurun_out/s2_san_${tool}_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s2_san_${tool}_pytest.txt; done
