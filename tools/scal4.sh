run() { n=$1; shift; tag=$1; shift; s=$(date +%s); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n "$@" > gpurun_out/v_$tag.json 2> gpurun_out/v_$tag.err; echo "$tag rc=$? $(( $(date +%s)-s ))s" >> gpurun_out/v_times.txt; }
run 2 d2
run 4 d4
CUDA_VISIBLE_DEVICES=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_v2_kernel -c 1 -o gpurun_out/ncu_conv1_2_n8 python tools/kbench.py 8 64 1024 1024 64 3 1 1 --ops fwd --bn-fused --iters 1 --warmup 1 > gpurun_out/ncu_conv.log 2>&1
echo "ncu rc=$?" >> gpurun_out/v_times.txt
