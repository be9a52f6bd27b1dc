timeout 200 python dbg_wgrad.py > gpurun_out/dbg.log 2>&1; echo dbg rc=$?
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "not full_size" -s > gpurun_out/gpu_tests.log 2>&1; echo tests rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench4.log 2>&1; echo bench rc=$?
