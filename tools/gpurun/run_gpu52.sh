export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm2|k_wgrad_bf16x6|k_xent" -c 5 -f -o gpurun_out/r1_dense_full3 $B > gpurun_out/g52_a.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g52_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/g52_d.log 2>&1
