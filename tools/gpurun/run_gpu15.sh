export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g15_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/g15_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g15_tests.log
timeout 600 python bench.py > gpurun_out/g15_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/g15_bench.log
timeout 600 python bench.py --cache-l1 --no-e2e > gpurun_out/g15_bench_l1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g15_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/g15_ncu_bench.log 2>&1
