# confirm the epilogue-group rule: parity (1 and 2 GPUs), key layers, bench at 1 and 2 GPUs
timeout 900 python -m pytest tests -m gpu -x -q -rs > gpurun_out/gputests5.log 2>&1; echo "tests $?" > gpurun_out/c_status.txt
for sh in "8 18 2048 2048 64 3 2 1" "8 64 1024 1024 64 3 1 1" "8 64 1024 1024 128 3 2 1" "8 256 256 256 256 3 1 1"; do
  CUDA_VISIBLE_DEVICES=0 timeout 120 python tools/kbench.py $sh --ops fwd,bpx --bn-fused --flush --iters 20 --warmup 5 >> gpurun_out/epi_c.txt 2>&1
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/bc1.json 2> gpurun_out/bc1.err; echo "bench1 $?" >> gpurun_out/c_status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > gpurun_out/bc2.json 2> gpurun_out/bc2.err; echo "bench2 $?" >> gpurun_out/c_status.txt
