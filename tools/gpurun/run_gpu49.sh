export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py --shapes 100x256,256x256,256x48 > gpurun_out/g49_gemm.log 2>&1
