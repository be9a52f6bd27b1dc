export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g62_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g62_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g62_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g62_smoke.log
timeout 600 python bench.py > gpurun_out/g62_bench.log 2>&1
