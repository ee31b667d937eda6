timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.txt 2>&1; echo rc=$? >> gpurun_out/f2_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f2_gputest.txt 2>&1; echo rc=$? >> gpurun_out/f2_gputest.txt
timeout 600 python bench.py > gpurun_out/f2_bench_sk.json 2> gpurun_out/f2_bench_sk.err
timeout 600 python bench.py --net usk > gpurun_out/f2_bench_usk.json 2> gpurun_out/f2_bench_usk.err
timeout 600 python bench.py --net u > gpurun_out/f2_bench_u.json 2> gpurun_out/f2_bench_u.err
for k in crt_gemm_rw_kernel crt_chain3_kernel crt_certify2_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/f2_$k python tools/prof_run.py --size 1024 --steps 1 > gpurun_out/f2_ncu_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-tc > gpurun_out/f2_ncu_bench.log 2>&1
