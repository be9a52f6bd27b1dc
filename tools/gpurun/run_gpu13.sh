export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -s -x > gpurun_out/gpu_tests13.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench13.log 2>&1; echo bench rc=$?
