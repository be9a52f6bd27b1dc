export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm_variants.py -q -p no:cacheprovider -k "TMA" > gpurun_out/g54_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g54_tests.log
o=gpurun_out/g54_sweep.log; : > $o
for t in 0 1; do echo "== tma=$t" >> $o; DIGEST_SPMM_TMA=$t timeout 300 python tools/spmm_bench.py --mode 1 --widths 48,100,256 >> $o 2>&1; done
for t in 0 1; do echo "== M8 tma=$t" >> $o; DIGEST_SPMM_TMA=$t timeout 300 python tools/spmm_bench.py --parts 8 --mode 1 --widths 48,100,256 >> $o 2>&1; done
