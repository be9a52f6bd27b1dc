export PYTHONUNBUFFERED=1
for v in 0 2 3 4; do DIGEST_SPMM_V=$v timeout 200 python tools/spmm_bench.py --widths 256 > gpurun_out/sb10_v$v.log 2>&1; done
timeout 300 python tools/spmm_bench.py --widths 256,128,100,64,48,32,16,8 > gpurun_out/sb10_widths.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "not full_size" -x > gpurun_out/gpu_tests10.log 2>&1; echo tests rc=$?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench10.log 2>&1; echo bench rc=$?
