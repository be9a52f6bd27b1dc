export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g59_repeat.jsonl; : > $o
for i in 1 2 3; do timeout 600 python bench.py --steps 40 --no-e2e 2>/dev/null | grep '^{' >> $o; done
