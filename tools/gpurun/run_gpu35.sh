export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g35_sweep.log; : > $o
for v in 0 2 3 4 5; do echo "== w100 v25=$v" >> $o; DIGEST_SPMM_V25=$v timeout 200 python tools/spmm_bench.py --widths 100 >> $o 2>&1; done
for v in 0 3 4 5; do echo "== M8 w100 v25=$v" >> $o; DIGEST_SPMM_V25=$v timeout 200 python tools/spmm_bench.py --parts 8 --widths 100 >> $o 2>&1; done
for v in 0 1; do echo "== M8 w48 v12=$v" >> $o; DIGEST_SPMM_V12=$v timeout 200 python tools/spmm_bench.py --parts 8 --widths 48 >> $o 2>&1; done
