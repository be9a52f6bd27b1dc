export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "xent or trajectory" > gpurun_out/g42_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g42_parity.log
timeout 600 python bench.py > gpurun_out/g42_bench.log 2>&1
