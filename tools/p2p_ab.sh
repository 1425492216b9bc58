T="timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2"
$T --shape bloom-7b1 --batch 8 --ctx 512 --steps 10 --warmup 3 --no-cpu-baseline --hop p2p > gpurun_out/p2p_7b1.log 2>&1
$T --shape bloom-7b1 --batch 8 --ctx 512 --steps 10 --warmup 3 --no-cpu-baseline --hop nccl > gpurun_out/nccl_7b1.log 2>&1
$T --steps 10 --warmup 3 --no-cpu-baseline --hop p2p > gpurun_out/p2p_176b.log 2>&1
$T --steps 10 --warmup 3 --no-cpu-baseline --hop nccl > gpurun_out/nccl_176b.log 2>&1
