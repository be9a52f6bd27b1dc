export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g44_sweep.log; : > $o
for h in 0 1; do echo "== pfh=$h" >> $o; DIGEST_SPMM_PFH=$h timeout 200 python tools/spmm_bench.py --widths 256,100 >> $o 2>&1; done
for h in 0 1; do echo "== M8 pfh=$h" >> $o; DIGEST_SPMM_PFH=$h timeout 200 python tools/spmm_bench.py --parts 8 --widths 256,100 >> $o 2>&1; done
for h in 0 1; do echo "== reddit pfh=$h" >> $o; DIGEST_SPMM_PFH=$h timeout 300 python tools/spmm_bench.py --config reddit --widths 256 >> $o 2>&1; done
