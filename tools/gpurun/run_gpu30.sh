export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/g30_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g30_tests.log
timeout 600 python bench.py > gpurun_out/g30_bench.log 2>&1
timeout 600 python bench.py --config reddit > gpurun_out/g30_bench_reddit.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g30_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/g30_d.log 2>&1
