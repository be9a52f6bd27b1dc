export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g39_sweep.log; : > $o
echo "== new addressing" >> $o; timeout 200 python tools/spmm_bench.py --widths 256,100,48 >> $o 2>&1
echo "== M8 new addressing" >> $o; timeout 200 python tools/spmm_bench.py --parts 8 --widths 256,100,48 >> $o 2>&1
