nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k gemm -x > gpurun_out/gemm_tests.log 2>&1; echo gemm rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "not full_size" > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.log 2>&1; echo bench rc=$?
