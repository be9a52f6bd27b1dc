export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bf16_store.py tests/test_gpu_peer.py -v -p no:cacheprovider > gpurun_out/g27_bf16.log 2>&1; echo "rc=$?" >> gpurun_out/g27_bf16.log
timeout 600 python bench.py > gpurun_out/g27_bench.log 2>&1
timeout 600 python bench.py --loopback 8 --sync-interval 1 --steps 10 --store-bf16 > gpurun_out/g27_bench_bf16.log 2>&1
