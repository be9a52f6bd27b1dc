export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g34_sweep.log; : > $o
for v in 0 2; do echo "== reddit v=$v" >> $o; DIGEST_SPMM_V=$v timeout 300 python tools/spmm_bench.py --config reddit --widths 256 >> $o 2>&1; done
for v in 0 2; do echo "== M8 v=$v" >> $o; DIGEST_SPMM_V=$v timeout 300 python tools/spmm_bench.py --parts 8 --widths 256 >> $o 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spmm_variants.py -q -x -p no:cacheprovider -k "layer or trajectory or fresh or w256" > gpurun_out/g34_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g34_parity.log
timeout 600 python bench.py > gpurun_out/g34_bench.log 2>&1
