timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --sources 8 > gpurun_out/bench2.log 2>&1; echo "rc=$?"
tail -c 1500 gpurun_out/bench2.log
