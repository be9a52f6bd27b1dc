for sl in 0 128 64 32; do
  DIGEST_SPMM_SLAB=$sl timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e > gpurun_out/bench8_$sl.log 2>&1; echo slab $sl rc=$?
  DIGEST_SPMM_SLAB=$sl timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_spmm -s 24 -c 24 --csv --log-file gpurun_out/spmm8_$sl.csv python bench.py --steps 1 --warmup 1 --no-e2e > /dev/null 2>&1; echo ncu rc=$?
done
