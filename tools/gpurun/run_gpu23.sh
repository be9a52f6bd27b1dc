export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_async.py -v -p no:cacheprovider > gpurun_out/g23_peer.log 2>&1; echo "rc=$?" >> gpurun_out/g23_peer.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "layer or trajectory or fresh" > gpurun_out/g23_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g23_parity.log
timeout 600 python bench.py > gpurun_out/g23_bench.log 2>&1
