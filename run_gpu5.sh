timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "not full_size" -x > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench5.log 2>&1; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 80 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu rc=$?
