export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "optimizers or cuda_graph" > gpurun_out/g45_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g45_tests.log
o=gpurun_out/g45_graph.jsonl; : > $o
for c in cora flickr arxiv products; do for gflag in "" "--graph"; do timeout 600 python bench.py --config $c $gflag --steps 20 2>gpurun_out/g45_err_$c.log | grep '^{' >> $o; done; done
