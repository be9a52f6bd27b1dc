export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g36_sweep.log; : > $o
for v in 0 1; do echo "== arxiv v32=$v" >> $o; DIGEST_SPMM_V32=$v timeout 300 python bench.py --config arxiv --no-e2e --steps 20 2>/dev/null | grep '^{' >> $o; done
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/g36_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g36_tests.log
for c in products reddit flickr; do timeout 600 python bench.py --config $c > gpurun_out/g36_bench_$c.log 2>&1; done
