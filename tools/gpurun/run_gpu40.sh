export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k full_size -s > gpurun_out/g40_full.log 2>&1; echo "rc=$?" >> gpurun_out/g40_full.log
