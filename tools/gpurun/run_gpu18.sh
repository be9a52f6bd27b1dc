export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g18_spmm.log; : > $o
for cfg in "products 1" "products 8" "reddit 1"; do set -- $cfg
for grid in 1 0; do for slab in 0 32 64 128; do
  echo "== $1 parts=$2 grid=$grid slab=$slab" >> $o
  DIGEST_SPMM_GRID=$grid DIGEST_SPMM_SLAB=$slab timeout 300 python tools/spmm_bench.py --config $1 --parts $2 --widths 256,100,48 >> $o 2>&1
done; done; done
