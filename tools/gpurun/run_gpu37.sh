export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_spmm -c 3 -f -o gpurun_out/r1_spmm_full2 $B > gpurun_out/g37_a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm2 -c 2 -f -o gpurun_out/r1_gemm_full2 $B > gpurun_out/g37_b.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g37_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/g37_d.log 2>&1
