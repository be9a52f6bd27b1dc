export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/g53_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g53_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g53_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g53_smoke.log
timeout 600 python bench.py > gpurun_out/g53_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g53_ref.log 2>&1
for c in reddit arxiv flickr; do timeout 600 python bench.py --config $c > gpurun_out/g53_bench_$c.log 2>&1; done
