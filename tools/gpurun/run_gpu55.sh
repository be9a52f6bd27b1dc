export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_variants.py -q -p no:cacheprovider -k "TMA" > gpurun_out/g55_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g55_tests.log
echo "== tma=1 w256" > gpurun_out/g55_sweep.log; DIGEST_SPMM_TMA=1 timeout 300 python tools/spmm_bench.py --mode 1 --widths 256 >> gpurun_out/g55_sweep.log 2>&1
