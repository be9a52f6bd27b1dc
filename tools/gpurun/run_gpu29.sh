export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g29_sweep.log; : > $o
for h in 1 2 0; do for cs in 0 1; do
 echo "== hints=$h stream_out=$cs" >> $o; DIGEST_SPMM_HINTS=$h DIGEST_SPMM_STREAM_OUT=$cs timeout 200 python tools/spmm_bench.py --widths 256,100,48 >> $o 2>&1
done; done
