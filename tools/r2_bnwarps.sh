# staged BN kernels: 12 vs 15 consumer warps (source edited on the box)
export CUDA_VISIBLE_DEVICES=0
F=paper_1903_06681_b200/csrc/bn.cu
for W in 12 15 12 15; do
  sed -i "s/constexpr int kBnWarps = [0-9]*,/constexpr int kBnWarps = $W,/" $F
  python -m paper_1903_06681_b200.build > /dev/null
  echo "== $W consumer warps"
  for sh in "8 64 1024 1024" "8 256 256 256" "8 512 64 64"; do timeout 120 python tools/bn_bench.py $sh --iters 50; done
done
sed -i "s/constexpr int kBnWarps = [0-9]*,/constexpr int kBnWarps = 15,/" $F
python -m paper_1903_06681_b200.build > /dev/null
timeout -k 10 600 python -m pytest tests/test_gpu_network.py tests/test_gpu_edge.py tests/test_loopback.py -m gpu -q 2>&1 | tail -1
