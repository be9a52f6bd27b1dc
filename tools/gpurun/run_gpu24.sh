export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "layer or trajectory or fresh" > gpurun_out/g24_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g24_parity.log
o=gpurun_out/g24_sweep.log; : > $o
for v in 0 1 2; do echo "== w100 v25=$v" >> $o; DIGEST_SPMM_V25=$v timeout 200 python tools/spmm_bench.py --widths 100 >> $o 2>&1; done
timeout 600 python bench.py > gpurun_out/g24_bench.log 2>&1
