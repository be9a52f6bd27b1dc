export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g57_sweep.log; : > $o
for v in 0 5 6 7; do echo "== w48 v12=$v" >> $o; DIGEST_SPMM_V12=$v timeout 200 python tools/spmm_bench.py --widths 48 >> $o 2>&1; done
for v in 0 5 6 7; do echo "== M8 w48 v12=$v" >> $o; DIGEST_SPMM_V12=$v timeout 200 python tools/spmm_bench.py --parts 8 --widths 48 >> $o 2>&1; done
timeout 600 python -m pytest tests/test_gpu_spmm_variants.py -q -p no:cacheprovider -k "w48" > gpurun_out/g57_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g57_tests.log
