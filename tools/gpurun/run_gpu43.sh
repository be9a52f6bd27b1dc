export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
o=gpurun_out/g43_loopback.jsonl; : > $o
for m in 2 4 8; do for mode in sync async; do timeout 600 python bench.py --loopback $m --mode $mode --steps 20 2>/dev/null | grep '^{' >> $o; done; done
for m in 2 4 8; do timeout 600 python bench.py --config reddit --loopback $m --steps 20 2>/dev/null | grep '^{' >> $o; done
for m in 4 8; do timeout 600 python bench.py --config arxiv --loopback $m --steps 20 2>/dev/null | grep '^{' >> $o; done
for m in 2 4; do timeout 600 python bench.py --config flickr --loopback $m --steps 20 2>/dev/null | grep '^{' >> $o; done
timeout 600 python bench.py --config cora --loopback 2 --steps 20 2>/dev/null | grep '^{' >> $o
timeout 600 python bench.py --config cora --steps 20 2>/dev/null | grep '^{' >> $o
