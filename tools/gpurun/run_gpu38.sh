export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g38_sweep.log; : > $o
for x in 0 1; do echo "== xr=$x" >> $o; DIGEST_SPMM_XR=$x timeout 200 python tools/spmm_bench.py --widths 256,100,48 >> $o 2>&1; done
for x in 0 1; do echo "== M8 xr=$x" >> $o; DIGEST_SPMM_XR=$x timeout 200 python tools/spmm_bench.py --parts 8 --widths 256,100,48 >> $o 2>&1; done
