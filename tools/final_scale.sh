# final round-1 scaling: bench.py at 1, 2, 4 GPUs as the driver launches it
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/fs_1.json 2> gpurun_out/fs_1.err; echo "n1 $?" > gpurun_out/fs_status.txt
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n > gpurun_out/fs_$n.json 2> gpurun_out/fs_$n.err; echo "n$n $?" >> gpurun_out/fs_status.txt
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/fs_ref2.json 2> gpurun_out/fs_ref2.err; echo "ref2 $?" >> gpurun_out/fs_status.txt
