export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_spmm_variants.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "variant or layer or trajectory" > gpurun_out/g51_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g51_tests.log
timeout 600 python bench.py --no-e2e > gpurun_out/g51_bench.log 2>&1
