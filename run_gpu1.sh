set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "not full_size" > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.log 2>&1; echo bench rc=$?
