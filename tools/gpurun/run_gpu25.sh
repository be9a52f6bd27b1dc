export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g25_sweep.log; : > $o
for h in 1 0; do for v in 0 1; do for mb in 0 4; do
 echo "== w48 pfh=$h v12=$v mb=$mb" >> $o; DIGEST_SPMM_PFH=$h DIGEST_SPMM_V12=$v DIGEST_SPMM_MB=$mb timeout 200 python tools/spmm_bench.py --widths 48 >> $o 2>&1
done; done; done
for h in 1 0; do echo "== M8 pfh=$h" >> $o; DIGEST_SPMM_PFH=$h timeout 200 python tools/spmm_bench.py --parts 8 --widths 48,100,256 >> $o 2>&1; done
