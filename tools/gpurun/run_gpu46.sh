export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g46_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g46_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g46_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g46_smoke.log
timeout 600 python bench.py > gpurun_out/g46_bench.log 2>&1
timeout 600 python bench.py --config cora --graph --steps 20 > gpurun_out/g46_cora_graph.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g46_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/g46_d.log 2>&1
