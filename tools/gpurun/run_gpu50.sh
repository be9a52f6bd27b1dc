export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py --shapes 100x256,256x256,48x256 > gpurun_out/g50_gemm.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo_grad.py -q -x -p no:cacheprovider -k "gemm or layer or trajectory or g_halo or full_size" > gpurun_out/g50_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g50_parity.log
