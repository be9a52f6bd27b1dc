export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g33_sweep.log; : > $o
for v in 0 1 2 3 4 5; do echo "== w256 v=$v" >> $o; DIGEST_SPMM_V=$v timeout 200 python tools/spmm_bench.py --widths 256 >> $o 2>&1; done
for mb in 4 5 6; do echo "== w256 v=0 mb=$mb" >> $o; DIGEST_SPMM_MB=$mb timeout 200 python tools/spmm_bench.py --widths 256 >> $o 2>&1; done
for v in 0 1 2; do for mb in 0 4; do echo "== w100 v25=$v mb=$mb" >> $o; DIGEST_SPMM_MB=$mb DIGEST_SPMM_V25=$v timeout 200 python tools/spmm_bench.py --widths 100 >> $o 2>&1; done; done
