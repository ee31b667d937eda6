timeout 600 python tools/scratch/x_exactness.py > gpurun_out/n_xstats.json 2> gpurun_out/n_xstats.err
for k in crt_gemm2_kernel crt_certify2_kernel crt_chain3_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/n_$k python tools/prof_run.py --size 1024 --steps 1 > gpurun_out/n_$k.log 2>&1
done
