export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g61_gemm.log; : > $o
for rb in 0 1; do echo "== resident_b=$rb" >> $o; DIGEST_GEMM_RESIDENT_B=$rb timeout 300 python tools/gemm_bench.py --shapes 48x256,256x48 >> $o 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo_grad.py -q -x -p no:cacheprovider -k "gemm or layer or trajectory or g_halo" > gpurun_out/g61_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g61_parity.log
