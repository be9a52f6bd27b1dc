export PYTHONUNBUFFERED=1
for v in 0 1 2 3 4 5; do DIGEST_SPMM_V=$v timeout 200 python tools/spmm_bench.py --widths 256 > gpurun_out/sb_v$v.log 2>&1; done
for h in 0 1; do for sl in 0 64 32; do DIGEST_SPMM_HINTS=$h DIGEST_SPMM_SLAB=$sl DIGEST_SPMM_V=2 timeout 200 python tools/spmm_bench.py --widths 256 > gpurun_out/sb_h${h}_s$sl.log 2>&1; done; done
timeout 300 python tools/spmm_bench.py --widths 256,128,100,64,48,32,16,8 > gpurun_out/sb_widths.log 2>&1
DIGEST_SPMM_V=2 timeout 300 ncu --set full --clock-control none -k regex:k_spmm -s 1 -c 1 -o gpurun_out/spmm256_v2 python tools/spmm_bench.py --widths 256 --iters 1 > /dev/null 2>&1
DIGEST_SPMM_V=2 DIGEST_SPMM_SLAB=32 timeout 300 ncu --set full --clock-control none -k regex:k_spmm -s 8 -c 1 -o gpurun_out/spmm256_slab32 python tools/spmm_bench.py --widths 256 --iters 1 > /dev/null 2>&1
echo done
