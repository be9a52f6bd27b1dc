export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "normalized or bf16" > gpurun_out/g60_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g60_tests.log
