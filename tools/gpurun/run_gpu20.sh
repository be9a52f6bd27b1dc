export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_async.py -v -x -p no:cacheprovider > gpurun_out/g20_async.log 2>&1; echo "rc=$?" >> gpurun_out/g20_async.log
