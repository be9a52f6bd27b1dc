export PYTHONUNBUFFERED=1
for v in 0 1 2; do DIGEST_SPMM_V25=$v timeout 200 python tools/spmm_bench.py --widths 100 > gpurun_out/sb14_v25_$v.log 2>&1; done
for v in 0 1 2 3 4; do DIGEST_SPMM_V12=$v timeout 200 python tools/spmm_bench.py --widths 48 > gpurun_out/sb14_v12_$v.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 900 -s -k "layer or fresh or full_size_products or trajectory" > gpurun_out/gpu_tests14.log 2>&1; echo tests rc=$?
