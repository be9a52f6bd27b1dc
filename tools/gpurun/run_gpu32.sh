export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g32_gemm.log; : > $o
for c in 1 0; do echo "== 2cta=$c" >> $o; DIGEST_GEMM_2CTA=$c timeout 300 python tools/gemm_bench.py --shapes 100x256,48x256,256x256 >> $o 2>&1; done
