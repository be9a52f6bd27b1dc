export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g31_sweep.log; : > $o
for hr in 0 32768 65536 98304 131072 196608; do
 echo "== hot_rows=$hr" >> $o; DIGEST_HOT_ROWS=$hr timeout 200 python tools/spmm_bench.py --widths 256,100 >> $o 2>&1
done
for hr in 0 49152 98304; do echo "== M8 hot_rows=$hr" >> $o; DIGEST_HOT_ROWS=$hr timeout 200 python tools/spmm_bench.py --parts 8 --widths 256 >> $o 2>&1; done
for hr in 0 98304; do echo "== reddit hot_rows=$hr" >> $o; DIGEST_HOT_ROWS=$hr timeout 300 python tools/spmm_bench.py --config reddit --widths 256,48 >> $o 2>&1; done
