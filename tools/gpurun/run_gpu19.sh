export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/g19_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g19_tests.log
timeout 600 python bench.py > gpurun_out/g19_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/g19_bench.log
timeout 600 python bench.py --config reddit --no-e2e > gpurun_out/g19_bench_reddit.log 2>&1
