# 1x1 stride-2 forward through the gathered pixels: parity, then the ResNet projection layers
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_conv.py -m gpu -q -x > gpurun_out/sub2_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/sub2_tests.log
for s in "64 1024 14 14 2048 1 2 0" "64 256 56 56 512 1 2 0" "64 512 28 28 1024 1 2 0" "64 256 56 56 128 1 2 0" "64 512 28 28 256 1 2 0" "64 1024 14 14 512 1 2 0"; do timeout 120 python tools/kbench.py $s --flush --iters 10; done
timeout -k 10 600 python bench.py --workload resnet50_n64 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/sub2_resnet.json 2> gpurun_out/sub2_resnet.err; echo "resnet $?"
