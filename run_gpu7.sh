timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e > gpurun_out/bench7.log 2>&1; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_spmm -s 5 -c 5 --csv --log-file gpurun_out/spmm7.csv python bench.py --steps 1 --warmup 1 --no-e2e > /dev/null 2>&1; echo ncu rc=$?
timeout 300 python -m pytest tests -m gpu -q -p no:cacheprovider -k "layer or trajectory" -x > gpurun_out/gpu_tests7.log 2>&1; echo tests rc=$?
