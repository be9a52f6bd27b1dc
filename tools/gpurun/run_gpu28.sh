export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g28_gemm.log; : > $o
for sa in 0 1; do echo "== single_arrive=$sa" >> $o; DIGEST_GEMM_SINGLE_ARRIVE=$sa timeout 300 python tools/gemm_bench.py --shapes 100x256,256x256,48x256,256x48 >> $o 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gemm or layer" > gpurun_out/g28_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g28_parity.log
