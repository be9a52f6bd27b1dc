export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_spmm_variants.py -q -p no:cacheprovider > gpurun_out/g26_variants.log 2>&1; echo "rc=$?" >> gpurun_out/g26_variants.log
o=gpurun_out/g26_sweep.jsonl; : > $o
for n in 1 5 10 20; do for m in async sync; do
 timeout 600 python bench.py --loopback 8 --sync-interval $n --mode $m --steps 20 2>/dev/null | grep '^{' >> $o
done; done
timeout 600 python bench.py --loopback 8 --fresh --steps 20 2>/dev/null | grep '^{' >> $o
timeout 600 python bench.py --loopback 4 --config reddit --sync-interval 10 --steps 20 2>/dev/null | grep '^{' >> $o
timeout 600 python bench.py --loopback 4 --config reddit --fresh --steps 20 2>/dev/null | grep '^{' >> $o
timeout 600 python bench.py --steps 20 > gpurun_out/g26_bench.log 2>&1
