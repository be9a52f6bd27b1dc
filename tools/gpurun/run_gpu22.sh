export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g22_sweep.log; : > $o
for mb in 0 4 6; do
for v in 0 1 2 3 4; do echo "== w48 v12=$v mb=$mb" >> $o; DIGEST_SPMM_MB=$mb DIGEST_SPMM_V12=$v timeout 200 python tools/spmm_bench.py --widths 48 >> $o 2>&1; done
for v in 0 1 2; do echo "== w100 v25=$v mb=$mb" >> $o; DIGEST_SPMM_MB=$mb DIGEST_SPMM_V25=$v timeout 200 python tools/spmm_bench.py --widths 100 >> $o 2>&1; done
done
