export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --share-gpu --steps 12 --warmup 3 > gpurun_out/g47_share2.log 2>&1; echo "rc=$?" >> gpurun_out/g47_share2.log
timeout 900 $TR --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --share-gpu --steps 12 --warmup 3 --graph > gpurun_out/g47_share4_graph.log 2>&1; echo "rc=$?" >> gpurun_out/g47_share4_graph.log
