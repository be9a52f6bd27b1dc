for sl in 0 128 64 32; do
  DIGEST_SPMM_SLAB=$sl timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e > gpurun_out/bench_slab$sl.log 2>&1; echo slab $sl rc=$?
done
DIGEST_SPMM_SLAB=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 2 -c 1 -o gpurun_out/spmm256_full python bench.py --steps 1 --warmup 1 --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncufull rc=$?
DIGEST_SPMM_SLAB=64 timeout 600 ncu --set full --clock-control none -k regex:k_spmm -s 3 -c 1 -o gpurun_out/spmm64slab_full python bench.py --steps 1 --warmup 1 --no-e2e > gpurun_out/ncu_full2.log 2>&1; echo ncufull2 rc=$?
