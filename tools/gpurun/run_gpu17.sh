export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29511 bench.py --gpus 2 --share-gpu --steps 5 --warmup 3 --no-e2e > gpurun_out/g17_share2.log 2>&1; echo "rc=$?" >> gpurun_out/g17_share2.log
timeout 900 $TR --nproc-per-node 4 --master-port 29512 bench.py --gpus 4 --share-gpu --steps 4 --warmup 3 --mode sync > gpurun_out/g17_share4.log 2>&1; echo "rc=$?" >> gpurun_out/g17_share4.log
for c in reddit arxiv flickr; do timeout 600 python bench.py --config $c --no-e2e --steps 10 > gpurun_out/g17_$c.log 2>&1; done
