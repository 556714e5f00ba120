# flattened 1x1 layers as [npix/8][8] images (16 x 8 tiles = 128 consecutive pixels, paired tiles)
export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/flat8_tests.log 2>&1; echo "tests $?"; tail -3 gpurun_out/flat8_tests.log
for s in "64 1024 14 14 2048 1 2 0" "64 512 7 7 2048 1 1 0" "64 2048 7 7 512 1 1 0" "64 1024 14 14 256 1 1 0" "64 256 14 14 1024 1 1 0" "64 256 56 56 64 1 1 0" "64 64 56 56 256 1 1 0"; do timeout 120 python tools/kbench.py $s --flush --iters 10; done
timeout -k 10 600 python bench.py --workload resnet50_n64 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/flat8_resnet.json 2> gpurun_out/flat8_resnet.err; echo "resnet $?"
