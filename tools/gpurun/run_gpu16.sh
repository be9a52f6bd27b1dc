export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer.py -v -x -p no:cacheprovider > gpurun_out/g16_peer.log 2>&1; echo "rc=$?" >> gpurun_out/g16_peer.log
