export CUDA_VISIBLE_DEVICES=0
python -m paper_1903_06681_b200.build > /dev/null
for sh in "8 256 256 256" "8 128 512 512" "8 512 128 128" "8 64 1024 1024"; do timeout 120 python tools/bn_bench.py $sh --iters 50; done
