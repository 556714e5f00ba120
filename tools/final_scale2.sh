# round-1 closing scaling run at HEAD (wgrad 256-filter tiles): bench.py at 1, 2, 4 GPUs as the driver launches it,
# plus one ncu --set full capture of wgrad_v2 on a 256-filter-tile layer (conv4_2 backward-filter, N=8)
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/fs_1.json 2> gpurun_out/fs_1.err; echo "n1 $?" > gpurun_out/fs_status.txt
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n > gpurun_out/fs_$n.json 2> gpurun_out/fs_$n.err; echo "n$n $?" >> gpurun_out/fs_status.txt
done
CUDA_VISIBLE_DEVICES=0 timeout 240 ncu --set full --clock-control none --import-source on -k regex:wgrad_v2_kernel -c 1 -o gpurun_out/ncu_wgrad_conv4_2_n8 python tools/kbench.py 8 512 128 128 512 3 1 1 --ops bpw --iters 1 --warmup 1 > gpurun_out/ncu_w42.log 2>&1; echo "w42 $?" >> gpurun_out/fs_status.txt
