export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python bench.py --cache-l1 --no-e2e > gpurun_out/g58_l1.log 2>&1
